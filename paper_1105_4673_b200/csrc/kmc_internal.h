// kmc_internal.h -- shared declarations of the CUDA kernels and the host runtime of
// libkmc_b200.so.  Product code; shares nothing with oracle/.
//
// Data layout in HBM: the lattice is bit-packed CELL-MAJOR.  One uint64 word
// holds one coarse cell (q_x*q_y <= 64 sites, local site s = ly*q_x + lx, bit s) of one bit-plane:
//   adsdes*:  plane 0 = occupied
//   zgb*:     plane 0 = CO, plane 1 = O        (vacant = neither)
// Words are stored [plane][storage row sy][replica r][cell column cx]; storage rows are the
// rank's owned cell rows, plus one ghost cell row above (sy = 0) and below (sy = My_local+1)
// when a 2D lattice is split over ranks (ghost = 1).  A row across all replicas is contiguous,
// so a halo exchange moves one contiguous block per plane.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kmc {

constexpr int kMaxClass = 32;
constexpr int kLogBuckets = 91;      // buckets j of the table-driven log
constexpr int kLogTab = 257;         // lookup entries: bucket of (mantissa bits 51..44 t, halved?) at t + halved

// Slot types, used by the host rate table.
enum SlotType { T_ADS = 0, T_DES = 1, T_HOP = 2, T_COADS = 3, T_O2ADS = 4, T_RCO = 5, T_RO = 6, T_COHOP = 7, T_OHOP = 8 };

struct Geo {
    int ndim, qx, qy, nsite;
    int Mx, My_local, R, ghost;      // cells per row, owned cell rows, replicas (local), ghost rows?
    int row_offset;                  // global cell row of owned row 0
    int rep_offset;                  // global replica of local replica 0
    long long M_global;              // cells per replica (global)
    int shN;                         // q_x*(q_y-1): bit offset of the last row
    uint64_t valid, col0, colL, row0, rowL;
    uint64_t notcol0, notcolL, notrow0, notrowL;   // valid & ~(...): kept in the param bank, not registers
};

struct SubstepArgs {
    Geo g;
    uint64_t* plane0;
    uint64_t* plane1;
    uint32_t* wev;                   // cumulative events per owned cell [My_local][R][Mx]
    unsigned long long* ev_total;    // device event counter
    unsigned int* queue;             // [2] chunk counters of the persistent window kernel: window w uses [w & 1]
    int colour, C;
    double D;                        // window duration
    double inv_scale;                // 2^-F
    double inv_half, inv_R;          // 1/half, 1/R for fast_divmod in the cell locator
    uint32_t half;                   // active cells per (row, replica): Mx/2, or the nested count in 1D
    // f3 nested decomposition (R28): the window runs only the cells of the outer blocks (`nest_B`
    // cell rows in 2D, cells in 1D) of one outer colour.  nest = 0: off.  In 2D the active rows are
    // numbered block by block, nest_rows per block; nest_s = parity of the first local block
    // that is active.
    int refill_min;                  // parked finished lanes that trigger a warp's refill (>= 1)
    int nest, nest_B, nest_s;
    uint32_t nest_rows;
    double inv_nest_rows;
    uint32_t key0, key1;             // Philox key = seed
    uint32_t rk0[10], rk1[10];       // Philox round keys k + i*(W0, W1), i = 0..9 (warp-uniform)
    uint32_t w_lo, w_hi_tag;         // window id (tag EVT = 0 in bits 28..31)
    uint64_t rate[kMaxClass];        // u64 fixed-point class rates (R18)
    uint64_t hopz[4];                // ADSDES_DIFF: (z - n) x the hop rate of block n (uniform blocks, R31)
    int hop_fast;                    // every hop block (ADSDES_DIFF) / direction group (ZGB) has one rate
    const double2* logtab;           // log_spec lookup {c_j, L_j}, kLogTab entries in device
                                     // memory: c_j = 128/(j+91), L_j = -log(c_j) (host libm), entry i holding
                                     // the bucket j of the mantissas with t = mant >> 44 = i (not halved,
                                     // i <= 0x6A) or t = i - 1 (halved, i >= 0x6B); kept out of the parameters
    double lcoef[6];                 //   {1/7, -1/6, 1/5, 1/3, ln2_hi, ln2_lo} (exact hex literals)
    // fused halo exchange (SURVEY §8(e) "later option"): the window kernel mirrors every write to a
    // boundary-row or ghost-row word into the neighbour ranks' planes (peer pointers: other slabs on
    // the same device, or CUDA-IPC mappings of a peer GPU's planes over NVLink), so no separate
    // exchange runs between windows.  peer_up[0] == nullptr: off.
    uint64_t* peer_up[2];
    uint64_t* peer_dn[2];
    int peer_up_rows;                // the up neighbour's owned cell rows (its last row / bottom ghost)
    int group;                       // lanes per cell (spin flip): 0 auto, 1 lane-per-cell kernel, g = 2..32
                                     // (last: a field above would shift the 16-byte alignment of the round keys)
};

struct ObsArgs {
    Geo g;
    const uint64_t* plane0;
    const uint64_t* plane1;
    int nplanes, C;
    unsigned long long* out;         // [4 n_state][16 by_colour][16 nn ordered], then events, windows, time
    unsigned long long windows;      // written to out[37] / out[38] by one thread (host values at enqueue)
    double time;
    unsigned long long* acc;         // [kObsCounters + 1] self-cleaning accumulator + block ticket (zero between calls)
    const unsigned long long* ev_total;
};

constexpr int kObsCounters = 4 + 16 + 16;

struct CorrArgs {
    Geo g;
    const uint64_t* plane0;
    const uint64_t* plane1;
    int nplanes, state, rmax, do_y;
    unsigned long long* out;         // [2][rmax+1]: pair counts along x, then y
};
constexpr int kMaxCorrR = 1024;      // largest rmax of kmc_correlation
cudaError_t launch_correlation(const CorrArgs& a, cudaStream_t s);

// f1: coverage process (R30).  One sample = per-replica count of `state` sites over the owned cells.
struct SeriesArgs {
    Geo g;
    const uint64_t* plane0;
    const uint64_t* plane1;
    int nplanes, state;
    unsigned long long* out;         // [R local] counts of this sample (zeroed by the caller)
};
cudaError_t launch_series_count(const SeriesArgs& a, cudaStream_t s);
// statistics over samples [first, n) of a series [n][R] (counts; coverage = count / nsite_rep):
//   tot            <- sum of the counts (u64, exact)
//   acov[l], l = 0..L  <- sum over (i, r), first <= i < n - l, of (c_i - mean)(c_{i+l} - mean), c in coverage
//                     units (count / nsite_rep); one block per lag, fixed reduction order (deterministic)
//   hist[b]        <- number of (i, r) with floor(count * bins / (nsite_rep + 1)) = b
cudaError_t launch_series_total(const unsigned long long* series, long long first, long long n, int R,
                                unsigned long long* tot, cudaStream_t s);
cudaError_t launch_series_acov(const unsigned long long* series, long long first, long long n, int R, int L,
                               double nsite_rep, double mean, double* acov, cudaStream_t s);
cudaError_t launch_series_hist(const unsigned long long* series, long long first, long long n, int R,
                               long long nsite_rep, int bins, unsigned long long* hist, cudaStream_t s);

// kernels.cu
cudaError_t launch_substep(int kind, const SubstepArgs& a, long long nactive, cudaStream_t s);
cudaError_t launch_substep_tile(const SubstepArgs& a, cudaStream_t s);   // kmc_tile.cu (2D spin flip)
cudaError_t queue_slot_reset(const SubstepArgs& a, cudaStream_t s);
cudaError_t launch_observables(const ObsArgs& a, cudaStream_t s);
cudaError_t launch_pack(const Geo& g, const uint8_t* in, uint64_t* p0, uint64_t* p1, int nstates,
                        unsigned int* err, cudaStream_t s);
cudaError_t launch_unpack(const Geo& g, const uint64_t* p0, const uint64_t* p1, int nplanes,
                          uint8_t* out, cudaStream_t s);
cudaError_t launch_init_random(const Geo& g, uint64_t* p0, uint64_t* p1, uint64_t seed, const unsigned long long* thr,
                               int nthr, cudaStream_t s);
cudaError_t launch_check_packed(const uint64_t* p0, const uint64_t* p1, long long n, uint64_t valid,
                                unsigned int* err, cudaStream_t s);
cudaError_t launch_strip_loads(const Geo& g, const uint32_t* wev, const uint32_t* mark, unsigned long long* strips,
                               cudaStream_t s);
cudaError_t launch_cdf_partition(unsigned long long* loads, unsigned long long* cdf, long long M, int P, int granule,
                                 long long* out, cudaStream_t s);
cudaError_t launch_wait_flags(unsigned long long* flags, unsigned long long epoch, cudaStream_t s);
cudaError_t launch_signal_flags(unsigned long long* up_flags, unsigned long long* dn_flags, unsigned long long v,
                                cudaStream_t s);
cudaError_t launch_xor_rows(uint64_t* dst, const uint64_t* a, const uint64_t* b, long long n, cudaStream_t s);
cudaError_t launch_copy_words(unsigned long long* dst, const unsigned long long* src, int n, cudaStream_t s);
cudaError_t launch_copy_u64(uint64_t* dst, const uint64_t* src, long long n, cudaStream_t s);

}  // namespace kmc
