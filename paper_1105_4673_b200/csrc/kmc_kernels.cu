// kmc_kernels.cu -- sm_100a kernels of the fractional-step KMC hot path.
//
// substep_kernel: one window e^{D L^c} of eq.(exact).
//   ONE LANE OWNS ONE COARSE CELL.  The cell and its one-site halo live in registers as
//   64-bit bitboards (bit-packed cell-major layout, kmc_internal.h); per event the lane
//     1. derives every slot class's member mask by bit-sliced neighbour counting
//        (the class is the rate-table index of eq.(Arrhenius) P:963-968 / Table COrates),
//     2. lambda = sum_c popc(mask_c) * rate_c   (eq.(totalrate), exact u64)
//     3. draws Philox4x32-10(k, gid, window) and the exponential clock tau = -ln U / lambda
//        (table-driven FMA log), stops when t + tau >= D (R5),
//     4. picks class c with prob popc*rate/lambda and a uniform member site of c
//        (eq.(skeleton)) with popc-based rank selection, and
//     5. applies the event as XORs on the planes (partner sites outside the cell go to
//        the halo boards, written back once per window with atomicXor of the delta).
//   No tensor cores: this is not a contraction.  See DESIGN.md §8 for why a lane (not a
//   warp) owns a cell: the per-event chain is serial, so 32 independent cells per warp
//   give 32x the issue efficiency of a warp-cooperative scan.  The event steps are in
//   kmc_device.cuh: event_step (generic, every model; also used by the tile kernel of
//   kmc_tile.cu), event_step_hop (diffusion, n-major hop blocks, R31; KIND 4) and
//   event_step_zgb_grouped (ZGB with one rate per direction group; KINDs 5, 6, 8).  Every 2D
//   variant is also built for 8 x 8 cells with the shape as a compile-time constant (SQ = 8).
// substep_group_kernel: the same window with g lanes per cell for windows with few active cells
//   (small lattices): the g lanes draw g consecutive events in parallel, then run them in order.
// observables_kernel (a8): integer counts, order-free, one launch per observation.
// correlation_kernel, series_*_kernel (f1): pair counts; the coverage process and its statistics.
// strip / cdf kernels (f4), init_random_kernel (R32), pack / unpack (uint8 site-major <->
// bit-packed cell-major), exchange helpers (flags, XOR rows) for the multi-GPU slabs.
#include "kmc_device.cuh"

#ifndef GROUP_SPEC
#define GROUP_SPEC 1   // lane-group kernel, spin flip: speculative event application (see group_window)
#endif

#include <cassert>
#include <cstdint>
#include <cstdlib>

// KMC_BOUNDS (debug builds, KMC_NVCC_FLAGS=-DKMC_DEBUG_BOUNDS): kmc_device.cuh

namespace kmc {

// ---------------------------------------------------------------------------------------------
// Lane-queue window kernel.
//
// Work distribution: the active cells of the colour are numbered 0..nactive-1 (row-major over
// (row, replica, column pair)); warp w owns the contiguous chunk [w*chunk, (w+1)*chunk).  Each
// lane runs one cell at a time; when its cell's window ends (clock past D or lambda = 0) the lane
// writes the cell back and takes the next unclaimed cell of the warp's chunk (ballot + popc, no
// atomics).  This keeps the 32 lanes busy although cells execute Poisson-distributed numbers of
// events -- with one static cell per lane a warp would run max-over-lanes iterations.
// ---------------------------------------------------------------------------------------------
struct CellLoc {
    uint32_t iC, iW, iE, iN, iS;      // word indices of the cell and its 4 neighbours (one plane)
    uint32_t sy;                      // storage row of the cell (owned rows are 1..My_local with ghosts)
    uint32_t iev;                     // index into the per-cell event counters
    uint32_t gid32;                   // global cell id (Philox counter word 1, R17)
};

// Active-cell number t -> cell location.  All indices fit 32 bits (kmc_create enforces < 2^32
// cells in total, and a plane holds at most that many words plus two ghost rows).
template <int NDIM, bool NEST>
__device__ __forceinline__ CellLoc locate(const SubstepArgs& a, uint32_t t) {
    const Geo& g = a.g;
    uint32_t rest, j, rowsel, r;
    if ((a.half & (a.half - 1u)) == 0u) {      // warp-uniform: half a power of two -> shift / mask
        j = t & (a.half - 1u);                  // (+0.6 % at dt = 0.01, where the refill is 37 % of the work)
        rest = t >> (31 - __clz(a.half));
    } else {
        fast_divmod(t, a.half, a.inv_half, rest, j);
    }
    if (g.R == 1) { rowsel = rest; r = 0; }
    else fast_divmod(rest, (uint32_t)g.R, a.inv_R, rowsel, r);
    uint32_t cy, cx;
    if (NDIM == 1) {
        cy = 0;
        if (NEST) {               // f3: pair j of the active outer blocks (B/2 pairs per block)
            uint32_t bb, i;
            fast_divmod(j, a.nest_rows, a.inv_nest_rows, bb, i);
            cx = (2 * bb + a.nest_s) * a.nest_B + 2 * i + a.colour;
        } else {
            cx = 2 * j + a.colour;
        }
    } else {
        uint32_t y0 = 0;          // first local row of the active outer block (f3), else 0
        if (NEST) {
            uint32_t bb, i;
            fast_divmod(rowsel, a.nest_rows, a.inv_nest_rows, bb, i);
            y0 = (2 * bb + a.nest_s) * a.nest_B;
            rowsel = i;
        }
        if (a.C == 2) {
            cy = y0 + rowsel;
            cx = 2 * j + ((a.colour + g.row_offset + cy) & 1);
        } else {
            cy = y0 + 2 * rowsel + (a.colour >> 1);
            cx = 2 * j + (a.colour & 1);
        }
    }
    const uint32_t gy = g.row_offset + cy;
    const uint32_t rowlen = (uint32_t)g.R * g.Mx;
    const int sy = (int)cy + g.ghost;
    int syN = sy - 1, syS = sy + 1;
    if (!g.ghost) {
        if (syN < 0) syN += g.My_local;
        if (syS >= g.My_local) syS -= g.My_local;
    }
    const uint32_t cxW = cx == 0 ? g.Mx - 1 : cx - 1;
    const uint32_t cxE = cx == (uint32_t)g.Mx - 1 ? 0 : cx + 1;
    const uint32_t rbase = r * g.Mx;
    const uint32_t base = (uint32_t)sy * rowlen + rbase;
    CellLoc L;
    L.sy = (uint32_t)sy;
    L.iC = base + cx;
    L.iW = base + cxW;
    L.iE = base + cxE;
    L.iN = (uint32_t)syN * rowlen + rbase + cx;
    L.iS = (uint32_t)syS * rowlen + rbase + cx;
    L.iev = cy * rowlen + rbase + cx;
    L.gid32 = (uint32_t)((unsigned long long)(g.rep_offset + r) * (unsigned long long)g.M_global +
                         (unsigned long long)gy * g.Mx + cx);
    KMC_BOUNDS(cx < (uint32_t)g.Mx && r < (uint32_t)g.R && cy < (uint32_t)g.My_local);
    KMC_BOUNDS(L.iC < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen && L.iW < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen &&
               L.iE < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen && L.iN < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen &&
               L.iS < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen && L.iev < (uint32_t)g.My_local * rowlen);
    return L;
}

// Fused exchange (PEER): mirror a modification of word `col` of storage row `row` into the
// neighbour slabs.  Rows: 0 = top ghost (= up's last owned row), 1 = first owned (= up's bottom
// ghost), My = last owned (= down's top ghost), My+1 = bottom ghost (= down's first owned row).
// Full-word stores go to ghost copies (no other writer of that word in this window); XOR deltas are
// system-scope atomics (the target may sit in a peer GPU's memory).
__device__ __forceinline__ void mirror_word(const SubstepArgs& a, int p, uint32_t row, uint32_t col, uint64_t v,
                                            bool is_xor) {
    const uint32_t rowlen = (uint32_t)a.g.R * a.g.Mx;
    const uint32_t My = (uint32_t)a.g.My_local, Mu = (uint32_t)a.peer_up_rows;
    uint64_t* tgt = nullptr;
    if (row == 0) tgt = a.peer_up[p] + (size_t)Mu * rowlen + col;
    else if (row == 1) tgt = a.peer_up[p] + (size_t)(Mu + 1) * rowlen + col;
    else if (row == My) tgt = a.peer_dn[p] + col;
    else if (row == My + 1) tgt = a.peer_dn[p] + (size_t)rowlen + col;
    if (!tgt) return;
    if (is_xor) atomicXor_system((unsigned long long*)tgt, (unsigned long long)v);
    else *tgt = v;
}

// One lane's cell: the closure in registers (a3) and its write-back (a6).
//   load: locate active cell c, its word and the four neighbour words per plane -> P, halo boards
//   store: the cell word once per window (+ the halo deltas of hop / pair events, XOR-merged into
//          the neighbour words: same-colour closures are disjoint, R6, so one writer per bit), the
//          per-cell event counter (RED) and the lane's event sum
template <int KIND, int NDIM, bool MH, bool NEST, bool PEER, int SQ = 0>
struct Cell {
    static constexpr int NP = Model<KIND, NDIM>::NP;
    uint64_t P[NP] = {}, h[NP][4] = {};   // zero until the first load: idle lanes step on a consistent empty cell
    uint32_t gid32 = 0, k = 0, iCcur = 0;
    uint32_t wrap = 0;   // hop / pair models: which neighbour indices wrap (W, E, N, S), for the store
    uint32_t srow = 0;   // PEER: storage row of the current cell
    double tclock = 0.0;

    __device__ __forceinline__ void load(const SubstepArgs& a, uint64_t* const* planes, uint32_t c) {
        const Geo& g = a.g;
        const CellLoc L = locate<NDIM, NEST>(a, c);
        gid32 = L.gid32;
        iCcur = L.iC;
        if constexpr (PEER) srow = L.sy;
        if constexpr (KIND != 0)
            wrap = (L.iW > L.iC ? 1u : 0u) | (L.iE < L.iC ? 2u : 0u) | (L.iN > L.iC ? 4u : 0u) | (L.iS < L.iC ? 8u : 0u);
        k = 0;
        tclock = 0.0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const uint64_t* pl = planes[p];
            P[p] = pl[L.iC];
            halo_from_words<MH, SQ>(g, pl[L.iW], pl[L.iE], NDIM == 2 ? pl[L.iN] : 0, NDIM == 2 ? pl[L.iS] : 0, h[p], NDIM == 2);
        }
    }

    __device__ __forceinline__ void store(const SubstepArgs& a, uint64_t* const* planes, unsigned long long& evsum,
                                          bool& peer_wrote) {
        const Geo& g = a.g;
        if (k == 0) return;
        if constexpr (KIND == 0) {   // spin flip writes only its own word: no second locate
            planes[0][iCcur] = P[0];
            if constexpr (PEER) {
                const uint32_t rl = (uint32_t)g.R * g.Mx;
                if (srow == 1 || srow == (uint32_t)g.My_local) {
                    mirror_word(a, 0, srow, iCcur - srow * rl, P[0], false);
                    peer_wrote = true;
                }
            }
            atomicAdd(&a.wev[iCcur - (uint32_t)g.ghost * ((uint32_t)g.R * g.Mx)], k);
            evsum += k;
            return;
        }
        // neighbour indices from the cell's own index and its wrap bits (no second locate)
        const uint32_t rowlen = (uint32_t)g.R * g.Mx;
        CellLoc L;
        L.iC = iCcur;
        L.iW = (wrap & 1u) ? iCcur + (uint32_t)(g.Mx - 1) : iCcur - 1u;
        L.iE = (wrap & 2u) ? iCcur - (uint32_t)(g.Mx - 1) : iCcur + 1u;
        L.iN = (wrap & 4u) ? iCcur + (uint32_t)(g.My_local - 1) * rowlen : iCcur - rowlen;
        L.iS = (wrap & 8u) ? iCcur - (uint32_t)(g.My_local - 1) * rowlen : iCcur + rowlen;
        L.iev = iCcur - (uint32_t)g.ghost * rowlen;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            uint64_t* pl = planes[p];
            pl[L.iC] = P[p];
            if (KIND != 0) {
                // halo deltas.  Our halo bits of the neighbour words are written by no other cell
                // in this window (same-colour closures are disjoint, R6), so re-reading them gives
                // the window-start values; the XOR touches only those bits (order-free).
                uint64_t hW, hE, hN, hS;
                halo_split<MH>(g, h[p], hW, hE, hN, hS);
                const int qx = SQ > 0 ? SQ : g.qx, shN = SQ > 0 ? SQ * (SQ - 1) : g.shN;
                const uint64_t dW = hW ^ ((pl[L.iW] >> (qx - 1)) & g.col0);
                const uint64_t dE = hE ^ ((pl[L.iE] << (qx - 1)) & g.colL);
                if (dW) atomicXor((unsigned long long*)&pl[L.iW], (unsigned long long)(dW << (qx - 1)));
                if (dE) atomicXor((unsigned long long*)&pl[L.iE], (unsigned long long)(dE >> (qx - 1)));
                uint64_t dN = 0, dS = 0;
                if (NDIM == 2) {
                    dN = hN ^ ((pl[L.iN] >> shN) & g.row0);
                    dS = hS ^ ((pl[L.iS] << shN) & g.rowL);
                    if (dN) atomicXor((unsigned long long*)&pl[L.iN], (unsigned long long)(dN << shN));
                    if (dS) atomicXor((unsigned long long*)&pl[L.iS], (unsigned long long)(dS >> shN));
                }
                if constexpr (PEER) {   // rows 0 / 1 / My / My+1 are shared with a neighbour slab
                    const uint32_t My = (uint32_t)g.My_local;
                    const uint32_t col = iCcur - srow * rowlen;
                    if (srow <= 2 || srow + 1 >= My) {
                        if (srow == 1 || srow == My) {
                            mirror_word(a, p, srow, col, P[p], false);
                            if (dW) mirror_word(a, p, srow, L.iW - srow * rowlen, dW << (g.qx - 1), true);
                            if (dE) mirror_word(a, p, srow, L.iE - srow * rowlen, dE >> (g.qx - 1), true);
                        }
                        if (dN) mirror_word(a, p, srow - 1, col, dN << g.shN, true);
                        if (dS) mirror_word(a, p, srow + 1, col, dS >> g.shN, true);
                        peer_wrote = true;
                    }
                }
            }
        }
        atomicAdd(&a.wev[L.iev], k);   // RED (no return): a plain += would stall on the load
        evsum += k;
    }
};

template <int KIND, int NDIM, int BS, int MINB, bool MH, bool NEST, bool PEER, int SQ = 0>
__global__ void __launch_bounds__(BS, MINB)
substep_kernel(const SubstepArgs a, const uint32_t nactive, const uint32_t chunk) {
    const Geo& g = a.g;
    const unsigned FULL = 0xffffffffu;
    // log_spec tables -> shared memory (lanes index them by their own bucket)
    __shared__ double2 s_logt[kLogTab];
    __shared__ __align__(16) uint8_t s_sel8[kSel8 + kDirTab];     // sel8 table + direction table
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) s_logt[i] = a.logtab[i];
    init_sel8(s_sel8);
    if constexpr (KIND != 0) init_dirtab(s_sel8, g);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.queue[(a.w_lo & 1u) ^ 1u] = 0u;   // the next window's counter
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long cbeg64 = (unsigned long long)warp * chunk;
    if (cbeg64 >= nactive) return;                                  // warp-uniform
    // The grid is persistent (about one wave): warp w starts on chunk w, then claims further chunks
    // of `chunk` cells from a global counter, so lanes never wait for a chunk boundary and there is
    // no wave-quantisation tail -- lanes idle only in the kernel's last cell-times.
    const unsigned long long pool0 = (unsigned long long)nwarps * chunk;   // first dynamic chunk
    uint32_t next = (uint32_t)cbeg64 + 32;                           // warp-uniform queue head
    uint32_t cend = (uint32_t)min(cbeg64 + chunk, (unsigned long long)nactive);
    bool pool_open = pool0 < nactive;
    uint64_t* planes[2] = {a.plane0, a.plane1};

    uint32_t ci = (uint32_t)cbeg64 + lane;
    bool have = ci < cend;
    Cell<KIND, NDIM, MH, NEST, PEER, SQ> cl;
    bool peer_wrote = false;
    unsigned long long evsum = 0;
    auto load = [&](uint32_t c) { cl.load(a, planes, c); };
    auto store = [&](uint32_t) { cl.store(a, planes, evsum, peer_wrote); };
    uint64_t* P = cl.P;
    uint64_t (*h)[4] = cl.h;
    uint32_t& k = cl.k;
    double& tclock = cl.tclock;
    const uint32_t& gid32 = cl.gid32;

    if (have) load(ci);
    // The event step is one branch-free basic block: lanes without a cell (queue exhausted) and
    // lanes whose window ended compute it too, with the update masked off, so the warp never
    // diverges inside the step and the scheduler can interleave its independent chains.
    // A lane whose window ends parks its finished cell (pend) until at least refill_min lanes are
    // parked (or none is running): the write-back + refill block costs the whole warp about half an
    // event step, so batching it trades a little lane idling for fewer executions.
    bool pend = false;
    const uint32_t refill_min = (uint32_t)a.refill_min;
    for (;;) {
        bool fin;
        if constexpr (KIND == 4) fin = event_step_hop<NDIM, MH, false, SQ>(a, P, h, k, tclock, gid32, have, s_logt, s_sel8);
        else if constexpr (KIND == 5 || KIND == 6)
            fin = event_step_zgb_grouped<KIND - 3, NDIM, MH, false, SQ>(a, P, h, k, tclock, gid32, have, s_logt, s_sel8);
        else if constexpr (KIND == 8)
            fin = event_step_zgb_grouped<7, NDIM, MH, false, SQ>(a, P, h, k, tclock, gid32, have, s_logt, s_sel8);
        else fin = event_step<KIND, NDIM, MH, false, SQ>(a, P, h, k, tclock, gid32, have, s_logt, s_sel8);
        pend = pend || fin;
        have = have && !fin;
        const unsigned fm = __ballot_sync(FULL, pend);
        if (fm && (__popc(fm) >= refill_min || !__any_sync(FULL, have))) {   // warp-uniform
            const bool fin = pend;
            pend = false;
            const uint32_t need = __popc(fm);
            const uint32_t rank = __popc(fm & ((1u << lane) - 1u));
            const uint32_t avail = cend > next ? cend - next : 0u;
            uint32_t nb = 0, nend = 0;
            bool claimed = false;
            if (need > avail && pool_open) {                       // warp-uniform: claim a chunk
                if (lane == 0) nb = atomicAdd(a.queue + (a.w_lo & 1u), chunk);
                const unsigned long long base = pool0 + __shfl_sync(FULL, nb, 0);
                claimed = base < nactive;
                pool_open = claimed;
                nb = (uint32_t)base;
                nend = claimed ? (uint32_t)min(base + chunk, (unsigned long long)nactive) : 0u;
            }
            if (fin) {
                store(ci);
                if (rank < avail) { ci = next + rank; have = true; }
                else { ci = nb + (rank - avail); have = claimed && ci < nend; }
                if (have) load(ci);
            }
            if (claimed) { next = nb + (need - avail); cend = nend; }
            else next += need;
            if (!__any_sync(FULL, have)) break;
        }
    }
    if constexpr (PEER) {
        if (peer_wrote) __threadfence_system();                    // peer writes visible before the signal
    }
    // event total: warp-aggregated
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evsum += __shfl_xor_sync(FULL, evsum, o);
    if (lane == 0 && evsum) atomicAdd(a.ev_total, evsum);
}

// ---------------------------------------------------------------------------------------------
// Lane-group window kernel for windows with few active cells (small lattices; SURVEY §7 step 8's
// lanes-per-cell parameter g): G lanes own one cell.  With one lane per cell such a window has
// too few warps to hide the latency of the serial per-event chain.  The serial part of an event
// (neighbour boards, lambda, tau, selection, update) depends on the previous event, the draws do
// not: the Philox block and E = -ln U of event k depend only on (k, gid, window) (R17).  So the G
// lanes of a group draw events k .. k+G-1 in parallel (lane j: event k+j; the next batch's draws
// are issued before this batch's serial steps, for ILP), then run the serial part of those events
// in order -- every lane of the group on the same cell state, draw j taken from lane j by shuffle
// -- until the cell's window ends (the first rejected draw, R5).  Same events, order and random
// numbers as substep_kernel: bit-identical results.
// ---------------------------------------------------------------------------------------------
// One window of the lane-group scheme for this thread's group (cell tid / G); returns the lane's
// event count (nonzero only in sub-lane 0, which writes the cell back).
template <int KIND, int NDIM, bool MH, int G, int SQ = 0>
__device__ __forceinline__ unsigned long long group_window(const SubstepArgs& a, uint32_t nactive, uint32_t tid,
                                                           const double2* s_logt, const uint8_t* s_sel8) {
    const unsigned FULL = 0xffffffffu;
    const uint32_t lane = threadIdx.x & 31u, sub = lane & (G - 1u), base = lane & ~(G - 1u);
    const uint32_t ci = tid / G;
    bool have = ci < nactive;
    uint64_t* planes[2] = {a.plane0, a.plane1};
    Cell<KIND, NDIM, MH, false, false, SQ> cl;
    if (have) cl.load(a, planes, ci);
    uint4 xd = philox_event(a, cl.k + sub, cl.gid32);
    double Ed = exp_variate(a, xd, s_logt);
    for (;;) {
        // a cell still running after this batch has accepted all G of its events: the next batch
        // is events k + G .. k + 2G - 1
        const uint4 xn = philox_event(a, cl.k + G + sub, cl.gid32);
        const double En = exp_variate(a, xn, s_logt);
        if constexpr (KIND == 0 && GROUP_SPEC) {
            // spin flip: the G events applied speculatively (each as if accepted), then the state
            // after the last accepted one kept: P before event j is snapshotted, the first rejected
            // event ends the window (R5) and the later ones are discarded
            uint64_t snap[G];
            double tsnap[G + 1];
            bool accj[G];
            tsnap[0] = cl.tclock;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                const int src = (int)(base | (uint32_t)j);
                uint4 xj;
                xj.x = 0u;
                xj.y = 0u;
                xj.z = __shfl_sync(FULL, xd.z, src);
                xj.w = __shfl_sync(FULL, xd.w, src);
                const double Ej = __hiloint2double(__shfl_sync(FULL, __double2hiint(Ed), src),
                                                   __shfl_sync(FULL, __double2loint(Ed), src));
                snap[j] = cl.P[0];
                event_step<KIND, NDIM, MH, true, SQ, true>(a, cl.P, cl.h, cl.k, cl.tclock, cl.gid32, have, s_logt,
                                                           s_sel8, xj, Ej, &accj[j]);
                tsnap[j + 1] = cl.tclock;
            }
            int nacc = 0;                                    // accepted events before the first rejection
            bool run = true;
#pragma unroll
            for (int j = 0; j < G; ++j) {
                run = run && accj[j];
                nacc += run ? 1 : 0;
            }
            uint64_t Pk = cl.P[0];
            double tk = tsnap[G];
#pragma unroll
            for (int j = G - 1; j >= 0; --j) {
                Pk = nacc == j ? snap[j] : Pk;
                tk = nacc == j ? tsnap[j] : tk;
            }
            cl.P[0] = Pk;
            cl.tclock = tk;
            cl.k += (uint32_t)nacc;
            have = have && nacc == G;
            if (!__any_sync(FULL, have)) break;
            xd = xn;
            Ed = En;
            continue;
        }
#pragma unroll
        for (int j = 0; j < G; ++j) {
            const int src = (int)(base | (uint32_t)j);
            uint4 xj;
            xj.x = 0u;
            xj.y = 0u;
            xj.z = __shfl_sync(FULL, xd.z, src);
            xj.w = __shfl_sync(FULL, xd.w, src);
            const double Ej = __hiloint2double(__shfl_sync(FULL, __double2hiint(Ed), src),
                                               __shfl_sync(FULL, __double2loint(Ed), src));
            bool fin;
            if constexpr (KIND == 4)
                fin = event_step_hop<NDIM, MH, true>(a, cl.P, cl.h, cl.k, cl.tclock, cl.gid32, have, s_logt, s_sel8, xj, Ej);
            else if constexpr (KIND == 5 || KIND == 6)
                fin = event_step_zgb_grouped<KIND - 3, NDIM, MH, true>(a, cl.P, cl.h, cl.k, cl.tclock, cl.gid32, have,
                                                                       s_logt, s_sel8, xj, Ej);
            else if constexpr (KIND == 8)
                fin = event_step_zgb_grouped<7, NDIM, MH, true>(a, cl.P, cl.h, cl.k, cl.tclock, cl.gid32, have, s_logt,
                                                                s_sel8, xj, Ej);
            else
                fin = event_step<KIND, NDIM, MH, true, SQ>(a, cl.P, cl.h, cl.k, cl.tclock, cl.gid32, have, s_logt, s_sel8, xj, Ej);
            have = have && !fin;
        }
        if (!__any_sync(FULL, have)) break;
        xd = xn;
        Ed = En;
    }
    unsigned long long evsum = 0;
    bool peer_wrote = false;
    if (sub == 0 && ci < nactive) cl.store(a, planes, evsum, peer_wrote);
    return evsum;
}

template <int KIND>
__device__ __forceinline__ void group_tables(const SubstepArgs& a, double2* s_logt, uint8_t* s_sel8) {
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) s_logt[i] = a.logtab[i];
    init_sel8(s_sel8);
    if constexpr (KIND != 0) init_dirtab(s_sel8, a.g);
}

__device__ __forceinline__ void add_events(unsigned long long evsum, unsigned long long* total) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evsum += __shfl_xor_sync(0xffffffffu, evsum, o);
    if ((threadIdx.x & 31u) == 0 && evsum) atomicAdd(total, evsum);
}

template <int KIND, int NDIM, bool MH, int G, int SQ = 0>
__global__ void __launch_bounds__(256)
substep_group_kernel(const SubstepArgs a, const uint32_t nactive) {
    __shared__ double2 s_logt[kLogTab];
    __shared__ __align__(16) uint8_t s_sel8[kSel8 + kDirTab];
    group_tables<KIND>(a, s_logt, s_sel8);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.queue[(a.w_lo & 1u) ^ 1u] = 0u;   // as substep_kernel
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    if ((tid & ~31u) / G >= nactive) return;                     // warp-uniform
    add_events(group_window<KIND, NDIM, MH, G, SQ>(a, nactive, tid, s_logt, s_sel8), a.ev_total);
}

// block size: the largest of 256 / 128 / 64 threads that still gives every SM two blocks (a 1024^2
// window is 8192 x 2 lanes: 64 blocks of 256 would leave 84 of the 148 SMs idle; 1024^2 at G = 2:
// 7.6e9 events/s with 256-thread blocks, 9.0e9 with 64 or 128).  KMC_GROUP_BS overrides.
template <int KIND, int NDIM, bool MH, int G, int SQ = 0>
static cudaError_t launch_group(const SubstepArgs& a, long long nactive, cudaStream_t s) {
    static int nsm = 0;
    if (nsm == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const long long threads = nactive * G;
    static const int bs_env = [] { const char* e = getenv("KMC_GROUP_BS"); return e ? atoi(e) : 0; }();
    int bs = 256;
    while (bs > 64 && (threads + bs - 1) / bs < 2LL * nsm) bs >>= 1;
    if (bs_env == 64 || bs_env == 128 || bs_env == 256) bs = bs_env;
    substep_group_kernel<KIND, NDIM, MH, G, SQ><<<(unsigned)((threads + bs - 1) / bs), bs, 0, s>>>(a, (uint32_t)nactive);
    return cudaGetLastError();
}

// resident CTAs per SM of one kernel instantiation (cached)
template <typename K>
static int resident_ctas(K kernel, int bs) {
    int dev = 0, nsm = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kernel, bs, 0) != cudaSuccess || per < 1) per = 1;
    return per * nsm;
}

template <int KIND, int NDIM, int MINB, bool MH, bool NEST, bool PEER = false, int BSZ = 256, int SQ = 0>
static cudaError_t launch_v(const SubstepArgs& a, long long nactive, cudaStream_t s) {
    constexpr int bs = BSZ;
    auto kern = substep_kernel<KIND, NDIM, bs, MINB, MH, NEST, PEER, SQ>;
    // persistent grid: one wave of resident warps, each starting on its own chunk of 32*8 cells
    static int cap = 0;                                            // per instantiation
    if (cap == 0) cap = resident_ctas(kern, bs);
    // chunk = 256 cells per claim; smaller windows get smaller chunks (multiples of 32, one cell per
    // lane at least) so that the grid still fills every resident warp slot
    const long long cap_warps = (long long)cap * (bs / 32);
    long long chunk = 32 * 8;
    while (chunk > 32 && (nactive + chunk - 1) / chunk < cap_warps) chunk -= 32;
    const long long want = (nactive + chunk - 1) / chunk;          // warps if every warp took one chunk
    const long long nwarps = want < cap_warps ? want : cap_warps;
    const unsigned nb = (unsigned)((nwarps * 32 + bs - 1) / bs);
    // no memset per window: the chunk counter is a.queue[w & 1], zeroed by the previous window
    // (queue_slot_reset); this kernel zeroes the other slot for the next window
    kern<<<nb, bs, 0, s>>>(a, (uint32_t)nactive, (uint32_t)chunk);
    return cudaGetLastError();
}

// a window that does not run substep_kernel (no active cells, or the tile kernel) zeroes the next
// window's chunk counter itself
cudaError_t queue_slot_reset(const SubstepArgs& a, cudaStream_t s) {
    return cudaMemsetAsync(a.queue + ((a.w_lo & 1u) ^ 1u), 0, sizeof(unsigned int), s);
}

// resident lanes of substep_kernel's launch shape (one lane per cell at full occupancy)
template <int KIND, int NDIM, int MINB, bool MH>
static long long launch_cap_lanes() {
    static long long cap = 0;
    if (cap == 0) cap = (long long)resident_ctas(substep_kernel<KIND, NDIM, 256, MINB, MH, false, false>, 256) * 256;
    return cap;
}

// lanes per cell for a window of nactive cells, from the queue kernel's resident lanes (148 SMs x 4
// CTAs x 256 = 151552 on B200): G = 1 above cap/8 cells, 2 down to cap/64, else 4.  Measured on
// B200 (tools/group_sweep.sh, KMC_GROUP = 1 / 2 / 4, events/s, with the block sizes below): 2D
// 1024^2 (8192 cells per window) 6.0e9 / 9.0e9 / 8.4e9; 1D 65536, one replica (1024 cells,
// launch-bound) 7.4e7 / 7.9e7 / 7.95e7; 1D 1024 x 1000 replicas (16000 cells) 1.66e9 / 1.74e9 /
// 1.64e9; 1D 65536 x 64 replicas (65536 cells) 3.89e9 / 3.69e9 / 3.05e9.  G = 8..32 was slower
// everywhere: the redundant serial steps cost more issue slots than the extra warps hide latency.
static int group_size(long long nactive, long long cap_lanes) {
    static const int env = [] { const char* e = getenv("KMC_GROUP"); return e ? atoi(e) : 0; }();
    if (env >= 1) return env;
    return nactive * 64 <= cap_lanes ? 4 : nactive * 8 <= cap_lanes ? 2 : 1;
}

// 8 x 8 cells (every 2D bench workload): kernels built with the cell shape as a compile-time
// constant (shift amounts in the neighbour boards, the halo extraction and the write-back), 10
// instructions fewer per spin-flip event step; measured +1.0 % (Lie dt = 1), +1.2 % (Strang),
// +2.1 % (dt = 0.01), +5 % (the lane-group kernel at 1024^2).  KMC_SQ8=0 disables.
static bool sq8(const SubstepArgs& a) {
    static const int env = [] { const char* e = getenv("KMC_SQ8"); return e ? atoi(e) : 1; }();
    return env && a.g.qx == 8 && a.g.qy == 8;
}

template <int KIND, int NDIM>
static cudaError_t launch_t(const SubstepArgs& a, long long nactive, cudaStream_t s) {
    if (nactive <= 0) return queue_slot_reset(a, s);
    // launch shape experiments: KMC_LB=3 forces the 128-register build, KMC_LB=4 the 80-register one,
    // KMC_LB=6 the 80-register spin-flip build; KMC_MH=1 merged halo boards for spin flip
    static const int lb = [] { const char* e = getenv("KMC_LB"); return e ? atoi(e) : 0; }();
    static const int mh_env = [] { const char* e = getenv("KMC_MH"); return e ? atoi(e) : -1; }();
    // merged halo boards need disjoint first/last columns (and rows in 2D)
    const bool mh_ok = a.g.qx >= 2 && (NDIM == 1 || a.g.qy >= 2);
    if constexpr (KIND == 0) {
        // few active cells (small lattices): G lanes per cell (substep_group_kernel).  KMC_GROUP = G
        // forces a group size (1 = off)
        if (!a.nest && !a.peer_up[0]) {
            const int G = a.group ? a.group : group_size(nactive, launch_cap_lanes<KIND, NDIM, 4, false>());
            if (NDIM == 2 && sq8(a) && (G == 2 || G == 4))
                return G == 2 ? launch_group<KIND, NDIM, false, 2, 8>(a, nactive, s)
                              : launch_group<KIND, NDIM, false, 4, 8>(a, nactive, s);
            switch (G) {
            case 2: return launch_group<KIND, NDIM, false, 2>(a, nactive, s);
            case 4: return launch_group<KIND, NDIM, false, 4>(a, nactive, s);
            case 8: return launch_group<KIND, NDIM, false, 8>(a, nactive, s);
            case 16: return launch_group<KIND, NDIM, false, 16>(a, nactive, s);
            case 32: return launch_group<KIND, NDIM, false, 32>(a, nactive, s);
            default: break;
            }
        }
        // spin flip: the four separate (window-constant) halo boards save 8 logic ops per event and
        // measured 3 % faster at dt = 1; <= 64 registers (no spills) -> 4 CTAs of 256 per SM
        if (a.nest) return launch_v<KIND, NDIM, 4, false, true>(a, nactive, s);
        if (NDIM == 2 && a.peer_up[0]) return launch_v<KIND, NDIM, 4, false, false, NDIM == 2>(a, nactive, s);
        if (mh_ok && mh_env == 1) return launch_v<KIND, NDIM, 3, true, false>(a, nactive, s);
        if (lb == 6) return launch_v<KIND, NDIM, 3, false, false>(a, nactive, s);
        if (NDIM == 2 && sq8(a)) return launch_v<KIND, NDIM, 4, false, false, false, 256, 8>(a, nactive, s);
        return launch_v<KIND, NDIM, 4, false, false>(a, nactive, s);
    } else {
        // hop / pair models need the merged boards (qx, qy >= 2 is enforced at create).  Diffusion
        // (22 masks live) is fastest with <= 128 registers (2 CTAs/SM), ZGB (counts + rebuilt mask)
        // with <= 80 registers (3 CTAs/SM) -- measured on B200
        if (!mh_ok) return cudaErrorInvalidValue;
        if constexpr (KIND == 1) {
            // uniform hop blocks (R31): the block-walk step.  Launch shape measured on 8192^2 Strang:
            // 128-thread blocks (88 registers, 5 CTAs = 20 warps/SM) 3.20e10 events/s; 256 x 2 (94
            // registers, 16 warps) 3.01e10; 256 x 3 (80 registers, 24 warps) 2.90e10; 96 x 7 2.89e10
            static const int hlb = [] { const char* e = getenv("KMC_HOPLB"); return e ? atoi(e) : 5; }();
            if (a.hop_fast) {
                if (hlb == 5) {
                    if (a.nest) return launch_v<4, NDIM, 5, true, true, false, 128>(a, nactive, s);
                    if (NDIM == 2 && a.peer_up[0]) return launch_v<4, NDIM, 5, true, false, NDIM == 2, 128>(a, nactive, s);
                    if (NDIM == 2 && sq8(a)) return launch_v<4, NDIM, 5, true, false, false, 128, 8>(a, nactive, s);
                    return launch_v<4, NDIM, 5, true, false, false, 128>(a, nactive, s);
                }
                if (a.nest) return hlb == 2 ? launch_v<4, NDIM, 2, true, true>(a, nactive, s)
                                            : launch_v<4, NDIM, 3, true, true>(a, nactive, s);
                if (NDIM == 2 && a.peer_up[0])
                    return hlb == 2 ? launch_v<4, NDIM, 2, true, false, NDIM == 2>(a, nactive, s)
                                    : launch_v<4, NDIM, 3, true, false, NDIM == 2>(a, nactive, s);
                if (hlb == 7) return launch_v<4, NDIM, 7, true, false, false, 96>(a, nactive, s);
                return hlb == 2 ? launch_v<4, NDIM, 2, true, false>(a, nactive, s)
                     : hlb == 4 ? launch_v<4, NDIM, 4, true, false>(a, nactive, s)
                                : launch_v<4, NDIM, 3, true, false>(a, nactive, s);
            }
        }
        if constexpr (KIND == 2 || KIND == 3 || KIND == 7) {
            // equal rates within every direction group: the grouped step (KMC_ZGBFAST=0 disables)
            static const int zf = [] { const char* e = getenv("KMC_ZGBFAST"); return e ? atoi(e) : 1; }();
            if (a.hop_fast && zf) {
                constexpr int KG = KIND == 7 ? 8 : KIND + 3;
                // launch shape measured on zgb2d_32768 (after the table-driven member boards): 256 x 3
                // (<= 80 registers, no spill) 1.98e10 events/s; 256 x 4 (64 registers, 34-byte spill)
                // 1.91e10; 128 x 6 1.88e10.  KMC_ZGBLB=4 selects the 4-CTA build
                static const int zlb = [] { const char* e = getenv("KMC_ZGBLB"); return e ? atoi(e) : 3; }();
                if (zlb == 4 && !a.nest && !a.peer_up[0]) return launch_v<KG, NDIM, 4, true, false>(a, nactive, s);
                if (a.nest) return launch_v<KG, NDIM, 3, true, true>(a, nactive, s);
                if (NDIM == 2 && a.peer_up[0]) return launch_v<KG, NDIM, 3, true, false, NDIM == 2>(a, nactive, s);
                if (NDIM == 2 && sq8(a)) return launch_v<KG, NDIM, 3, true, false, false, 256, 8>(a, nactive, s);
                return launch_v<KG, NDIM, 3, true, false>(a, nactive, s);
            }
        }
        const bool big = (KIND == 1 && lb != 4) || lb == 3;
        if (a.nest) return big ? launch_v<KIND, NDIM, 2, true, true>(a, nactive, s)
                               : launch_v<KIND, NDIM, 3, true, true>(a, nactive, s);
        if (NDIM == 2 && a.peer_up[0])
            return big ? launch_v<KIND, NDIM, 2, true, false, NDIM == 2>(a, nactive, s)
                       : launch_v<KIND, NDIM, 3, true, false, NDIM == 2>(a, nactive, s);
        return big ? launch_v<KIND, NDIM, 2, true, false>(a, nactive, s)
                   : launch_v<KIND, NDIM, 3, true, false>(a, nactive, s);
    }
}

cudaError_t launch_substep(int kind, const SubstepArgs& a, long long nactive, cudaStream_t s) {
    const bool two = a.g.ndim == 2;
    switch (kind) {
    case 0: return two ? launch_t<0, 2>(a, nactive, s) : launch_t<0, 1>(a, nactive, s);
    case 1: return two ? launch_t<1, 2>(a, nactive, s) : launch_t<1, 1>(a, nactive, s);
    case 2: return two ? launch_t<2, 2>(a, nactive, s) : launch_t<2, 1>(a, nactive, s);
    case 3: return two ? launch_t<3, 2>(a, nactive, s) : launch_t<3, 1>(a, nactive, s);
    case 4: return two ? launch_t<7, 2>(a, nactive, s) : launch_t<7, 1>(a, nactive, s);   // ZGB_ODIFF
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------------
// a8: observables.  Counters (u64): [0..3] n_state, [4..19] by colour [c*4+s],
// [20..35] ordered nearest-neighbour bonds (x, x+e) for e in {+x, +y}: [20 + a*4 + b].
// ---------------------------------------------------------------------------------------------
// The kernel counts only the occupied states s, b >= 1 (per cell: popc of each plane, and of each
// plane AND the +x / +y neighbour board of each plane); the vacant entries follow from identities of
// the periodic lattice -- every site has exactly one +e neighbour and is the +e neighbour of exactly
// one site, so per direction sum_b nn_e[s][b] = N_s and sum_s nn_e[s][b] = N_b, and N_0 = sites -
// sum N_s (per colour likewise).  The last block applies them to this rank's sums; the identities
// are linear, so per-rank words (mod 2^64) still add up to the global counts under the NCCL
// all-reduce or the vgroup sum.  Memory: a warp reads 32 consecutive cells (coalesced), the +x word
// of lane l is lane l+1's own word (shuffle; lane 31 and row ends load it), and every lane keeps U
// cells' loads in flight (the grid-stride loop is otherwise latency-bound: round 1 measured
// ~1.3 TB/s on the 128 MiB target lattice).
// ---------------------------------------------------------------------------------------------
template <int NP, int NDIM, int SQ = 0>
__global__ void __launch_bounds__(256) observables_kernel(const ObsArgs a) {
    constexpr int U = 4;
    const unsigned FULL = 0xffffffffu;
    const Geo& g = a.g;
    __shared__ unsigned long long sh[kObsCounters];
    __shared__ bool last;
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    // occupied states only: n[s], by colour bc[col][s], ordered bonds nn[s][b] (s, b = plane index)
    uint32_t n[NP], bc[4][NP], nn[NP][NP];
#pragma unroll
    for (int s = 0; s < NP; ++s) {
        n[s] = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) bc[c][s] = 0;
#pragma unroll
        for (int b = 0; b < NP; ++b) nn[s][b] = 0;
    }
    const uint32_t rowlen = (uint32_t)g.R * g.Mx;
    const uint32_t ncell = (uint32_t)g.My_local * rowlen;
    const double inv_mx = 1.0 / (double)g.Mx, inv_r = 1.0 / (double)g.R;
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint64_t* planes[2] = {a.plane0, a.plane1};
    // counts of one cell from its planes P, the +x neighbour words E and the +y neighbour words S
    const int qx = SQ > 0 ? SQ : g.qx, shN = SQ > 0 ? SQ * (SQ - 1) : g.shN;   // SQ: compile-time 8 x 8 cells
    auto count = [&](const uint64_t* P, const uint64_t* E, const uint64_t* S, int col) {
        uint64_t Bx[NP], By[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            Bx[p] = ((P[p] >> 1) & g.notcolL) | ((E[p] << (qx - 1)) & g.colL);                  // sigma(x + e_x)
            By[p] = NDIM == 2 ? ((P[p] >> qx) | ((S[p] << shN) & g.rowL)) : 0ull;                // sigma(x + e_y)
        }
#pragma unroll
        for (int s = 0; s < NP; ++s) {
            const uint32_t c = __popcll(P[s]);
            n[s] += c;
#pragma unroll
            for (int cc = 0; cc < 3; ++cc)                        // colour C-1 is n minus the others
                if (cc + 1 < a.C) bc[cc][s] += col == cc ? c : 0u;
#pragma unroll
            for (int b = 0; b < NP; ++b)
                nn[s][b] += __popcll(P[s] & Bx[b]) + (NDIM == 2 ? __popcll(P[s] & By[b]) : 0u);
        }
    };
    if (g.Mx % (32 * U) == 0) {
        // fast path: every aligned block of 32 U cells lies in one row (of one replica): one locate per
        // block, lane l holds cells cx0 + 32 u + l; the +x word of lane 31 is lane 0's of the next u
        for (uint32_t base = warp * 32u * U; base < ncell; base += nwarps * 32u * U) {   // warp-uniform
            uint32_t rest, cx0, cy, r;
            fast_divmod(base, (uint32_t)g.Mx, inv_mx, rest, cx0);
            fast_divmod(rest, (uint32_t)g.R, inv_r, cy, r);
            const int sy = (int)cy + g.ghost;
            int syS = sy + 1;
            if (!g.ghost && syS >= g.My_local) syS -= g.My_local;
            const uint32_t iC0 = (uint32_t)sy * rowlen + r * g.Mx + cx0, iS0 = (uint32_t)syS * rowlen + r * g.Mx + cx0;
            const uint32_t gy = g.row_offset + cy, cx = cx0 + lane;     // cx parity is the same for every u
            const int col = a.C == 2 ? (NDIM == 1 ? (int)(cx & 1) : (int)((cx + gy) & 1)) : (int)(cx & 1) + 2 * (int)(gy & 1);
            // the word after the block: the next cell of the row, or its first cell (periodic wrap)
            const uint32_t iNext = cx0 + 32u * U == (uint32_t)g.Mx ? iC0 + 32u * U - (uint32_t)g.Mx : iC0 + 32u * U;
            KMC_BOUNDS(cx0 + 32u * U <= (uint32_t)g.Mx && iS0 + 32u * U <= (uint32_t)(g.My_local + 2 * g.ghost) * rowlen &&
                       iC0 + 32u * U <= (uint32_t)(g.My_local + 2 * g.ghost) * rowlen);
            uint64_t Pw[U][NP], Sw[U][NP], Nx[NP];
#pragma unroll
            for (int p = 0; p < NP; ++p) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    Pw[u][p] = planes[p][iC0 + 32u * u + lane];
                    Sw[u][p] = NDIM == 2 ? planes[p][iS0 + 32u * u + lane] : 0ull;
                }
                Nx[p] = lane == 31u ? planes[p][iNext] : 0ull;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                uint64_t E[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    const uint64_t dn = __shfl_down_sync(FULL, Pw[u][p], 1);
                    const uint64_t first = u + 1 < U ? __shfl_sync(FULL, Pw[u + 1 < U ? u + 1 : u][p], 0) : Nx[p];
                    E[p] = lane == 31u ? first : dn;
                }
                count(Pw[u], E, Sw[u], col);
            }
        }
    } else {
        // general path (short or odd rows): every lane locates its own cells
        for (uint32_t base = warp * 32u * U; base < ncell; base += nwarps * 32u * U) {   // warp-uniform
            uint64_t Pw[U][NP], Sw[U][NP];
            uint32_t iC[U], cxv[U];
            int col[U];
            bool ok[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t t = base + (uint32_t)u * 32u + lane;
                ok[u] = t < ncell;
                uint32_t rest = 0, cx = 0, cy = 0, r = 0;
                if (ok[u]) {
                    fast_divmod(t, (uint32_t)g.Mx, inv_mx, rest, cx);
                    fast_divmod(rest, (uint32_t)g.R, inv_r, cy, r);
                }
                const int sy = (int)cy + g.ghost;
                int syS = sy + 1;
                if (!g.ghost && syS >= g.My_local) syS -= g.My_local;
                iC[u] = (uint32_t)sy * rowlen + r * g.Mx + cx;
                cxv[u] = cx;
                const uint32_t iS = (uint32_t)syS * rowlen + r * g.Mx + cx;
                KMC_BOUNDS(!ok[u] || (iC[u] < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen &&
                                      iS < (uint32_t)(g.My_local + 2 * g.ghost) * rowlen));
                const uint32_t gy = g.row_offset + cy;
                col[u] = a.C == 2 ? (NDIM == 1 ? (int)(cx & 1) : (int)((cx + gy) & 1)) : (int)(cx & 1) + 2 * (int)(gy & 1);
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    Pw[u][p] = ok[u] ? planes[p][iC[u]] : 0ull;
                    Sw[u][p] = (NDIM == 2 && ok[u]) ? planes[p][iS] : 0ull;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                // the +x neighbour cell: the next lane's cell unless this is lane 31 or a row end (wrap)
                const bool own = ok[u] && (lane == 31u || cxv[u] == (uint32_t)g.Mx - 1);
                const uint32_t iE = cxv[u] == (uint32_t)g.Mx - 1 ? iC[u] + 1u - (uint32_t)g.Mx : iC[u] + 1u;
                uint64_t E[NP];
#pragma unroll
                for (int p = 0; p < NP; ++p) {
                    E[p] = __shfl_down_sync(FULL, Pw[u][p], 1);
                    if (own) E[p] = planes[p][iE];
                }
                count(Pw[u], E, Sw[u], col[u]);
            }
        }
    }
    // block sums (warp redux, one shared atomic per warp and counter), then one global atomic each
    auto put = [&](int idx, uint32_t v) {
        const uint32_t w = __reduce_add_sync(FULL, v);
        if (lane == 0 && w) atomicAdd(&sh[idx], (unsigned long long)w);
    };
#pragma unroll
    for (int s = 0; s < NP; ++s) {
        put(1 + s, n[s]);
#pragma unroll
        for (int cc = 0; cc < 4; ++cc) put(4 + cc * 4 + 1 + s, bc[cc][s]);
#pragma unroll
        for (int b = 0; b < NP; ++b) put(20 + (1 + s) * 4 + 1 + b, nn[s][b]);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x)
        if (sh[i]) atomicAdd(&a.acc[i], sh[i]);
    // the last block to finish completes the vacant entries, moves the totals to `out` (no memset /
    // copy launches per call) and leaves the accumulator and the ticket zero for the next call
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(&a.acc[kObsCounters], 1ull) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x) sh[i] = atomicExch(&a.acc[i], 0ull);
    __syncthreads();
    if (threadIdx.x == 0) {
        constexpr int NS = NP + 1;
        const unsigned long long z = NDIM;                         // +e bonds per site
        const unsigned long long sites = (unsigned long long)g.nsite * ncell;
        // cells per colour on this rank: 2 colours split every row; 4 colours: (cx & 1) + 2 (gy & 1)
        unsigned long long ccol[4] = {0, 0, 0, 0};
        const unsigned long long half_row = (unsigned long long)(g.Mx / 2) * g.R;
        if (a.C == 2) {
            ccol[0] = ccol[1] = half_row * g.My_local;
        } else {
            const unsigned long long ne = (unsigned long long)(g.My_local + ((g.row_offset & 1) == 0 ? 1 : 0)) / 2;
            ccol[0] = ccol[1] = half_row * ne;
            ccol[2] = ccol[3] = half_row * ((unsigned long long)g.My_local - ne);
        }
        for (int s = 1; s < NS; ++s) {                              // the last colour's sites per state
            unsigned long long v = 0;
            for (int cc = 0; cc + 1 < a.C; ++cc) v += sh[4 + cc * 4 + s];
            sh[4 + (a.C - 1) * 4 + s] = sh[s] - v;
        }
        unsigned long long nsum = 0;
        for (int s = 1; s < NS; ++s) nsum += sh[s];
        sh[0] = sites - nsum;
        for (int cc = 0; cc < 4; ++cc) {
            unsigned long long v = 0;
            for (int s = 1; s < NS; ++s) v += sh[4 + cc * 4 + s];
            sh[4 + cc * 4] = ccol[cc] * (unsigned long long)g.nsite - v;
        }
        for (int s = 1; s < NS; ++s) {                              // nn[s][0] and nn[0][s]
            unsigned long long rs = 0, cs = 0;
            for (int b = 1; b < NS; ++b) { rs += sh[20 + s * 4 + b]; cs += sh[20 + b * 4 + s]; }
            sh[20 + s * 4] = z * sh[s] - rs;
            sh[20 + s] = z * sh[s] - cs;
        }
        unsigned long long r0 = 0;
        for (int b = 1; b < NS; ++b) r0 += sh[20 + b];
        sh[20] = z * sh[0] - r0;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x) a.out[i] = sh[i];
    if (threadIdx.x == 0) {
        a.out[kObsCounters] = *(volatile const unsigned long long*)a.ev_total;
        a.out[kObsCounters + 1] = a.windows;
        a.out[kObsCounters + 2] = (unsigned long long)__double_as_longlong(a.time);
        a.out[kObsCounters + 3] = 0ull;
        a.acc[kObsCounters] = 0ull;
    }
}

// ---------------------------------------------------------------------------------------------
// f1: two-point correlation counts.  For a displacement r = a q + b along x (y), the partner of
// every site of a cell lies in the cells a and a+1 further along the axis; the partner board is
// assembled from those two words with shifts and column (row) masks and AND-ed with the cell's
// own state board.  Warp-reduced per r (redux.sync), then one shared and one global atomic.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint64_t state_board(const CorrArgs& a, long long idx) {
    const uint64_t p0 = a.plane0[idx];
    if (a.nplanes == 1) return a.state == 1 ? p0 : (a.g.valid & ~p0);
    const uint64_t p1 = a.plane1[idx];
    return a.state == 1 ? p0 : a.state == 2 ? p1 : (a.g.valid & ~(p0 | p1));
}

__global__ void __launch_bounds__(256) correlation_kernel(const CorrArgs a) {
    extern __shared__ unsigned long long sc[];            // [2][rmax+1]
    const Geo& g = a.g;
    const int R1 = a.rmax + 1;
    for (int i = threadIdx.x; i < 2 * R1; i += blockDim.x) sc[i] = 0;
    __syncthreads();
    const long long rowlen = (long long)g.R * g.Mx;
    const long long ncell = (long long)g.My_local * rowlen;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // warp-uniform trip count: every lane of a warp runs the same iterations (redux needs all 32)
    for (long long base = (long long)blockIdx.x * blockDim.x; base < ncell; base += stride) {
        const long long t = base + threadIdx.x;
        const bool ok = t < ncell;
        int cx = 0, r = 0, cy = 0;
        if (ok) {
            cx = (int)(t % g.Mx);
            const long long rest = t / g.Mx;
            r = (int)(rest % g.R);
            cy = (int)(rest / g.R);
        }
        const int sy = cy + g.ghost;
        const long long rb = (long long)r * g.Mx;
        const uint64_t A = ok ? state_board(a, (long long)sy * rowlen + rb + cx) : 0ull;
        // ---- along x ----
        {
            int aa = 0;
            uint64_t W0 = A, W1 = ok ? state_board(a, (long long)sy * rowlen + rb + (cx + 1) % g.Mx) : 0ull;
            for (int rr = 0, b = 0; rr < R1; ++rr) {
                uint64_t S;
                if (b == 0) S = W0;
                else {
                    const uint64_t lowcols = ((1ull << (g.qx - b)) - 1ull) * g.col0;   // columns < qx-b
                    S = ((W0 >> b) & lowcols) | ((W1 << (g.qx - b)) & (g.valid & ~lowcols));
                }
                const uint32_t v = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(A & S));
                if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sc[rr], (unsigned long long)v);
                if (++b == g.qx) {                           // next whole cell
                    b = 0;
                    ++aa;
                    W0 = W1;
                    W1 = ok ? state_board(a, (long long)sy * rowlen + rb + (cx + aa + 1) % g.Mx) : 0ull;
                }
            }
        }
        // ---- along y ----
        if (a.do_y) {
            auto rowidx = [&](int k) -> long long {           // storage row of the cell k rows below
                int yy = sy + k;
                if (!g.ghost) yy %= g.My_local;
                return (long long)yy * rowlen + rb + cx;
            };
            int aa = 0;
            uint64_t W0 = A, W1 = ok ? state_board(a, rowidx(1)) : 0ull;
            for (int rr = 0, b = 0; rr < R1; ++rr) {
                uint64_t S;
                if (b == 0) S = W0;
                else S = ((W0 >> (b * g.qx)) | (W1 << ((g.qy - b) * g.qx))) & g.valid;
                const uint32_t v = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(A & S));
                if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sc[R1 + rr], (unsigned long long)v);
                if (++b == g.qy) {
                    b = 0;
                    ++aa;
                    W0 = W1;
                    if (rr + 2 < R1) W1 = ok ? state_board(a, rowidx(aa + 1)) : 0ull;   // needed only if b > 0 follows
                }
            }
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 2 * R1; i += blockDim.x)
        if (sc[i]) atomicAdd(&a.out[i], sc[i]);
}

cudaError_t launch_correlation(const CorrArgs& a, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long ncell = (long long)a.g.My_local * a.g.R * a.g.Mx;
    long long nb = (ncell + 255) / 256;
    if (nb > 8LL * nsm) nb = 8LL * nsm;
    if (nb < 1) nb = 1;
    const size_t smem = (size_t)2 * (a.rmax + 1) * sizeof(unsigned long long);
    correlation_kernel<<<(unsigned)nb, 256, smem, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// f1: the coverage process C_t (Figs. path1D, autocorr1D, pdf2d, dynamics2d; P:1057-1062,
// P:1121-1127), recorded on the device at macro-step boundaries without a host round trip.
// series_count_kernel: per-replica number of `state` sites.  Cells are numbered [cy][r][cx], so a
// warp's lanes mostly share a replica: lanes are grouped by replica (match.any), each group
// reduced (redux.sync) and its leader does one u64 atomic.
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) series_count_kernel(const SeriesArgs a) {
    const Geo& g = a.g;
    const uint32_t rowlen = (uint32_t)g.R * g.Mx;
    const uint32_t ncell = (uint32_t)g.My_local * rowlen;
    const double inv_mx = 1.0 / (double)g.Mx, inv_r = 1.0 / (double)g.R;
    const uint32_t stride = gridDim.x * blockDim.x;
    // warp-uniform trip count (the group reductions need every lane of the warp)
    for (uint32_t base = blockIdx.x * blockDim.x; base < ncell; base += stride) {
        const uint32_t t = base + threadIdx.x;
        const bool ok = t < ncell;
        uint32_t rest = 0, cx = 0, cy = 0, r = 0;
        uint32_t cnt = 0;
        if (ok) {
            fast_divmod(t, (uint32_t)g.Mx, inv_mx, rest, cx);
            fast_divmod(rest, (uint32_t)g.R, inv_r, cy, r);
            const size_t idx = (size_t)(cy + (uint32_t)g.ghost) * rowlen + (size_t)r * g.Mx + cx;
            const uint64_t p0 = a.plane0[idx];
            const uint64_t p1 = a.nplanes > 1 ? a.plane1[idx] : 0ull;
            const uint64_t board = a.state == 1 ? p0 : a.state == 2 ? p1 : (g.valid & ~(p0 | p1));
            cnt = (uint32_t)__popcll(board);
        }
        const unsigned grp = __match_any_sync(0xffffffffu, ok ? r : 0xffffffffu);
        const uint32_t sum = __reduce_add_sync(grp, cnt);
        if (ok && (threadIdx.x & 31) == (unsigned)(__ffs(grp) - 1) && sum)
            atomicAdd(&a.out[r], (unsigned long long)sum);
    }
}

cudaError_t launch_series_count(const SeriesArgs& a, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long ncell = (long long)a.g.My_local * a.g.R * a.g.Mx;
    long long nb = (ncell + 255) / 256;
    if (nb > 8LL * nsm) nb = 8LL * nsm;
    if (nb < 1) nb = 1;
    series_count_kernel<<<(unsigned)nb, 256, 0, s>>>(a);
    return cudaGetLastError();
}

// sum of the counts of samples [first, n): one block, exact integer sum
__global__ void __launch_bounds__(256) series_total_kernel(const unsigned long long* __restrict__ ser, long long first,
                                                           long long n, int R, unsigned long long* tot) {
    __shared__ unsigned long long sh[8];
    unsigned long long acc = 0;
    const long long lo = first * R, hi = n * R;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += ser[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += sh[w];
        *tot = t;
    }
}

// acov[l] = sum_{r} sum_{i=first}^{n-1-l} (c_{i,r} - mean)(c_{i+l,r} - mean), c = count / nsite: one
// block per lag; each thread strides a fixed set of (i, r) pairs and the block tree-reduces in a
// fixed order, so the result is deterministic.
__global__ void __launch_bounds__(256) series_acov_kernel(const unsigned long long* __restrict__ ser, long long first,
                                                          long long n, int R, double nsite, double mean,
                                                          double* acov) {
    __shared__ double sh[256];
    const long long l = blockIdx.x;
    const long long m = (n - l - first) * R;            // pairs (i, r) with first <= i < n - l
    double acc = 0.0;
    for (long long j = threadIdx.x; j < m; j += blockDim.x) {
        const long long i0 = first * R + j;              // sample i = first + j / R, replica j % R
        const double a = (double)ser[i0] / nsite - mean;
        const double b = (double)ser[i0 + l * R] / nsite - mean;
        acc = __fma_rn(a, b, acc);
    }
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x >> 1; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) acov[l] = sh[0];
}

__global__ void __launch_bounds__(256) series_hist_kernel(const unsigned long long* __restrict__ ser, long long first,
                                                          long long n, int R, long long nsite, int bins,
                                                          unsigned long long* hist) {
    const long long lo = first * R, hi = n * R;
    for (long long i = lo + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long c = ser[i];
        const long long b = (long long)(c * (unsigned long long)bins / (unsigned long long)(nsite + 1));
        atomicAdd(&hist[b < bins ? b : bins - 1], 1ull);
    }
}

cudaError_t launch_series_total(const unsigned long long* ser, long long first, long long n, int R,
                                unsigned long long* tot, cudaStream_t s) {
    series_total_kernel<<<1, 256, 0, s>>>(ser, first, n, R, tot);
    return cudaGetLastError();
}

cudaError_t launch_series_acov(const unsigned long long* ser, long long first, long long n, int R, int L,
                               double nsite, double mean, double* acov, cudaStream_t s) {
    series_acov_kernel<<<(unsigned)(L + 1), 256, 0, s>>>(ser, first, n, R, nsite, mean, acov);
    return cudaGetLastError();
}

cudaError_t launch_series_hist(const unsigned long long* ser, long long first, long long n, int R, long long nsite,
                               int bins, unsigned long long* hist, cudaStream_t s) {
    const long long m = (n - first) * R;
    long long nb = (m + 255) / 256;
    if (nb > 1024) nb = 1024;
    if (nb < 1) nb = 1;
    series_hist_kernel<<<(unsigned)nb, 256, 0, s>>>(ser, first, n, R, nsite, bins, hist);
    return cudaGetLastError();
}

cudaError_t launch_observables(const ObsArgs& a, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long ncell = (long long)a.g.My_local * a.g.R * a.g.Mx;
    long long nb = (ncell + 255) / 256;
    if (nb > 4LL * nsm) nb = 4LL * nsm;
    if (nb < 1) nb = 1;
    const bool q8 = a.g.ndim == 2 && a.g.qx == 8 && a.g.qy == 8;
    if (a.nplanes == 1) {
        if (q8) observables_kernel<1, 2, 8><<<(unsigned)nb, 256, 0, s>>>(a);
        else if (a.g.ndim == 2) observables_kernel<1, 2><<<(unsigned)nb, 256, 0, s>>>(a);
        else observables_kernel<1, 1><<<(unsigned)nb, 256, 0, s>>>(a);
    } else {
        if (q8) observables_kernel<2, 2, 8><<<(unsigned)nb, 256, 0, s>>>(a);
        else if (a.g.ndim == 2) observables_kernel<2, 2><<<(unsigned)nb, 256, 0, s>>>(a);
        else observables_kernel<2, 1><<<(unsigned)nb, 256, 0, s>>>(a);
    }
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// pack / unpack between uint8 site-major [R][H_local][W] and the bit-packed planes.
// ---------------------------------------------------------------------------------------------
__global__ void pack_kernel(const Geo g, const uint8_t* __restrict__ in, uint64_t* p0, uint64_t* p1,
                            int nstates, unsigned int* err) {
    const long long ncell = (long long)g.My_local * g.R * g.Mx;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncell) return;
    const int cx = (int)(t % g.Mx);
    const long long rest = t / g.Mx;
    const int r = (int)(rest % g.R);
    const int cy = (int)(rest / g.R);
    const long long W = (long long)g.Mx * g.qx;
    const long long H = (long long)g.My_local * g.qy;
    uint64_t a = 0, b = 0;
    unsigned bad = 0;
    for (int ly = 0; ly < g.qy; ++ly) {
        const uint8_t* row = in + ((long long)r * H + (long long)cy * g.qy + ly) * W + (long long)cx * g.qx;
        for (int lx = 0; lx < g.qx; ++lx) {
            const unsigned v = row[lx];
            const int s = ly * g.qx + lx;
            if (v >= (unsigned)nstates) { bad = 1; continue; }
            a |= (uint64_t)(v == 1) << s;
            b |= (uint64_t)(v == 2) << s;
        }
    }
    const long long idx = ((long long)(cy + g.ghost) * g.R + r) * g.Mx + cx;
    p0[idx] = a;
    if (p1) p1[idx] = b;
    if (bad) atomicOr(err, 1u);
}

__global__ void unpack_kernel(const Geo g, const uint64_t* __restrict__ p0, const uint64_t* __restrict__ p1,
                              int nplanes, uint8_t* __restrict__ out) {
    const long long ncell = (long long)g.My_local * g.R * g.Mx;
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncell) return;
    const int cx = (int)(t % g.Mx);
    const long long rest = t / g.Mx;
    const int r = (int)(rest % g.R);
    const int cy = (int)(rest / g.R);
    const long long W = (long long)g.Mx * g.qx;
    const long long H = (long long)g.My_local * g.qy;
    const long long idx = ((long long)(cy + g.ghost) * g.R + r) * g.Mx + cx;
    const uint64_t a = p0[idx];
    const uint64_t b = nplanes > 1 ? p1[idx] : 0;
    for (int ly = 0; ly < g.qy; ++ly) {
        uint8_t* row = out + ((long long)r * H + (long long)cy * g.qy + ly) * W + (long long)cx * g.qx;
        for (int lx = 0; lx < g.qx; ++lx) {
            const int s = ly * g.qx + lx;
            row[lx] = (uint8_t)(((a >> s) & 1) | (((b >> s) & 1) << 1));
        }
    }
}

cudaError_t launch_pack(const Geo& g, const uint8_t* in, uint64_t* p0, uint64_t* p1, int nstates,
                        unsigned int* err, cudaStream_t s) {
    const long long ncell = (long long)g.My_local * g.R * g.Mx;
    if (ncell == 0) return cudaSuccess;
    pack_kernel<<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(g, in, p0, p1, nstates, err);
    return cudaGetLastError();
}

cudaError_t launch_unpack(const Geo& g, const uint64_t* p0, const uint64_t* p1, int nplanes,
                          uint8_t* out, cudaStream_t s) {
    const long long ncell = (long long)g.My_local * g.R * g.Mx;
    if (ncell == 0) return cudaSuccess;
    unpack_kernel<<<(unsigned)((ncell + 255) / 256), 256, 0, s>>>(g, p0, p1, nplanes, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// f4: workload histogram (eq.(wload)) per strip and the cdf re-partition (P:919-925,
// R29).  Strips: cell rows (2D, summed over columns and replicas) or cells (1D, over replicas).
// W(m) = wev(m) - mark(m) (u32 counters, wrap-safe difference).
// ---------------------------------------------------------------------------------------------
__global__ void strip_rows_kernel(const Geo g, const uint32_t* __restrict__ wev, const uint32_t* __restrict__ mark,
                                  unsigned long long* strips) {
    // one CTA per owned cell row: the row's R*Mx counters are contiguous
    const int cy = blockIdx.x;
    const long long n = (long long)g.R * g.Mx, base = (long long)cy * n;
    unsigned long long acc = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) acc += (uint32_t)(wev[base + i] - mark[base + i]);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    __shared__ unsigned long long part[32];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long t = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += part[w];
        atomicAdd(&strips[g.row_offset + cy], t);
    }
}

__global__ void strip_cells_kernel(const Geo g, const uint32_t* __restrict__ wev, const uint32_t* __restrict__ mark,
                                   unsigned long long* strips) {
    const int cx = blockIdx.x * blockDim.x + threadIdx.x;          // 1D: one thread per cell, over replicas
    if (cx >= g.Mx) return;
    unsigned long long acc = 0;
    for (int r = 0; r < g.R; ++r) acc += (uint32_t)(wev[(long long)r * g.Mx + cx] - mark[(long long)r * g.Mx + cx]);
    atomicAdd(&strips[cx], acc);
}

cudaError_t launch_strip_loads(const Geo& g, const uint32_t* wev, const uint32_t* mark, unsigned long long* strips,
                               cudaStream_t s) {
    if (g.ndim == 2) {
        if (g.My_local > 0) strip_rows_kernel<<<g.My_local, 256, 0, s>>>(g, wev, mark, strips);
    } else {
        strip_cells_kernel<<<(g.Mx + 255) / 256, 256, 0, s>>>(g, wev, mark, strips);
    }
    return cudaGetLastError();
}

// R29 rounding of one raw bound to the granule g (nearest multiple, ties up) and clamping
__device__ __forceinline__ long long round_clamp(long long x, long long prev, int l, int P, long long M, long long gr) {
    long long r = gr * ((2 * x + gr) / (2 * gr));
    r = r > prev + gr ? r : prev + gr;
    const long long hi = M - (long long)(P - l) * gr;
    return r < hi ? r : hi;
}

// One CTA: inclusive cdf of the M strip loads (segmented block scan), the P-1 raw bounds by binary
// search (min s+1 with P*cdf[s] >= l*S), rounding/clamping, and the imbalance (max group load x P / S)
// of the cdf partition and of the even split.  out = [bounds P+1 (i64)][imb_cdf, imb_even (f64)].
__global__ void __launch_bounds__(1024) cdf_partition_kernel(unsigned long long* loads, unsigned long long* cdf,
                                                             long long M, int P, int gr, long long* out) {
    __shared__ unsigned long long seg_sum[1024];
    const int t = threadIdx.x, nt = blockDim.x;
    const long long seg = (M + nt - 1) / nt;
    const long long a = (long long)t * seg, b = a + seg < M ? a + seg : M;
    unsigned long long acc = 0;
    for (long long i = a; i < b; ++i) acc += loads[i];
    seg_sum[t] = acc;
    __syncthreads();
    if (t == 0) {                                   // exclusive scan of the segment sums
        unsigned long long run = 0;
        for (int i = 0; i < nt; ++i) { const unsigned long long v = seg_sum[i]; seg_sum[i] = run; run += v; }
    }
    __syncthreads();
    acc = seg_sum[t];
    for (long long i = a; i < b; ++i) { acc += loads[i]; cdf[i] = acc; }
    __syncthreads();
    __threadfence_block();
    const unsigned long long S = cdf[M - 1];
    for (int l = 1 + t; l < P; l += nt) {           // raw bounds
        long long raw;
        if (S == 0) {
            raw = ((long long)l * M + P / 2) / P;
        } else {
            const unsigned long long thr = (unsigned long long)l * S;
            long long lo = 0, hi = M - 1;           // min s with P*cdf[s] >= thr (exists: P*S >= thr)
            while (lo < hi) {
                const long long mid = (lo + hi) >> 1;
                if ((unsigned long long)P * cdf[mid] >= thr) hi = mid; else lo = mid + 1;
            }
            raw = lo + 1;
        }
        out[l] = raw;
    }
    __syncthreads();
    if (t == 0) {
        auto load = [&](long long x, long long y) -> unsigned long long {
            return (y > 0 ? cdf[y - 1] : 0ull) - (x > 0 ? cdf[x - 1] : 0ull);
        };
        out[0] = 0;
        long long prev = 0;
        unsigned long long mx = 0, mx_even = 0, prev_even = 0;
        for (int l = 1; l <= P; ++l) {
            const long long bl = l < P ? round_clamp(out[l], prev, l, P, M, gr) : M;
            const long long be = l < P ? round_clamp(((long long)l * M + P / 2) / P, (long long)prev_even, l, P, M, gr) : M;
            const unsigned long long g1 = load(prev, bl), g2 = load((long long)prev_even, be);
            mx = g1 > mx ? g1 : mx;
            mx_even = g2 > mx_even ? g2 : mx_even;
            out[l] = bl;
            prev = bl;
            prev_even = (unsigned long long)be;
        }
        double* imb = reinterpret_cast<double*>(out + P + 1);
        imb[0] = S ? (double)mx * (double)P / (double)S : 1.0;
        imb[1] = S ? (double)mx_even * (double)P / (double)S : 1.0;
    }
}

cudaError_t launch_cdf_partition(unsigned long long* loads, unsigned long long* cdf, long long M, int P, int granule,
                                 long long* out, cudaStream_t s) {
    cdf_partition_kernel<<<1, 1024, 0, s>>>(loads, cdf, M, P, granule, out);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------------------------
// Fused exchange across GPUs: per-window neighbour synchronisation through flags in device memory
// (each rank's flags[0] is written by its up neighbour, flags[1] by its down neighbour, through
// CUDA-IPC mappings over NVLink).  A rank may start window e only when both neighbours have
// finished window e-1 (their peer writes into this rank are complete, and they no longer read the
// rows this window will write).  One thread.  A neighbour that does not arrive within kWaitNs
// (60 s of %globaltimer) does not hang the stream or trap the context: the kernel sets this rank's
// timeout word flags[2] and returns; kmc_device_errors / kmc_observables report it (the run after a
// timeout is not ordered and its results are void).
// ---------------------------------------------------------------------------------------------
constexpr unsigned long long kWaitNs = 60ull * 1000000000ull;

__global__ void wait_flags_kernel(unsigned long long* flags, unsigned long long epoch) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned long long a, b;
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(a) : "l"(flags));
        asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(b) : "l"(flags + 1));
        if (a >= epoch && b >= epoch) return;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > kWaitNs) { flags[2] = 1ull; return; }
        __nanosleep(200);
    }
}

__global__ void signal_flags_kernel(unsigned long long* up_flags, unsigned long long* dn_flags, unsigned long long v) {
    __threadfence_system();
    // I am my up neighbour's down neighbour (its flags[1]) and my down neighbour's up neighbour
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(up_flags + 1), "l"(v) : "memory");
    asm volatile("st.release.sys.global.u64 [%0], %1;" :: "l"(dn_flags), "l"(v) : "memory");
}

cudaError_t launch_wait_flags(unsigned long long* flags, unsigned long long epoch, cudaStream_t s) {
    wait_flags_kernel<<<1, 1, 0, s>>>(flags, epoch);
    return cudaGetLastError();
}

cudaError_t launch_signal_flags(unsigned long long* up_flags, unsigned long long* dn_flags, unsigned long long v,
                                cudaStream_t s) {
    signal_flags_kernel<<<1, 1, 0, s>>>(up_flags, dn_flags, v);
    return cudaGetLastError();
}

// validation of a bit-packed slab (kmc_set_config_packed): no bits outside the cell's sites, and in
// the two-plane models no site both CO and O
__global__ void check_packed_kernel(const uint64_t* __restrict__ p0, const uint64_t* __restrict__ p1,
                                    long long n, uint64_t valid, unsigned int* err) {
    unsigned bad = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const uint64_t a = p0[i];
        const uint64_t b = p1 ? p1[i] : 0ull;
        bad |= ((a | b) & ~valid) != 0 || (a & b) != 0;
    }
    // a plain store (every writer writes 1): err may be mapped pinned host memory (kmc_stage_config_packed)
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) *(volatile unsigned int*)err = 1u;
}

// ---------------------------------------------------------------------------------------------
// Random initial configuration (reading R32): site (x, y) of replica r takes
// state #{j : u >= T_j}, u = word 0 of Philox4x32-10((x, y, r, TAG_INIT << 28), seed).  One thread
// per owned cell writes the cell's bit-plane words; the state of a site depends on its global
// coordinates only (identical for any rank split).
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t philox_keyed_w0(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                    uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int rd = 0; rd < 10; ++rd) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c0;
}

__global__ void __launch_bounds__(256) init_random_kernel(const Geo g, uint64_t* p0, uint64_t* p1, uint32_t k0,
                                                          uint32_t k1, unsigned long long t0, unsigned long long t1,
                                                          int nthr) {
    const uint32_t rowlen = (uint32_t)g.R * g.Mx;
    const long long ncell = (long long)g.My_local * rowlen;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ncell;
         t += (long long)gridDim.x * blockDim.x) {
        const uint32_t cx = (uint32_t)(t % g.Mx);
        const uint32_t r = (uint32_t)((t / g.Mx) % g.R);
        const uint32_t cy = (uint32_t)(t / rowlen);
        const uint32_t y0 = (uint32_t)(g.row_offset + (int)cy) * (uint32_t)g.qy;
        uint64_t w0 = 0, w1 = 0;
        for (int ly = 0; ly < g.qy; ++ly)
            for (int lx = 0; lx < g.qx; ++lx) {
                const uint32_t u = philox_keyed_w0(cx * (uint32_t)g.qx + (uint32_t)lx, y0 + (uint32_t)ly,
                                                   (uint32_t)g.rep_offset + r, 2u << 28, k0, k1);
                const int st = (nthr > 0 && u >= t0 ? 1 : 0) + (nthr > 1 && u >= t1 ? 1 : 0);
                const uint64_t bit = 1ull << (ly * g.qx + lx);
                w0 |= st == 1 ? bit : 0ull;
                w1 |= st == 2 ? bit : 0ull;
            }
        const size_t idx = (size_t)(cy + (uint32_t)g.ghost) * rowlen + (size_t)r * g.Mx + cx;
        p0[idx] = w0;
        if (p1) p1[idx] = w1;
    }
}

cudaError_t launch_init_random(const Geo& g, uint64_t* p0, uint64_t* p1, uint64_t seed, const unsigned long long* thr,
                               int nthr, cudaStream_t s) {
    const long long ncell = (long long)g.My_local * g.R * g.Mx;
    if (ncell <= 0) return cudaSuccess;
    long long nb = (ncell + 255) / 256;
    if (nb > 148LL * 32) nb = 148LL * 32;
    init_random_kernel<<<(unsigned)nb, 256, 0, s>>>(g, p0, p1, (uint32_t)seed, (uint32_t)(seed >> 32),
                                                    nthr > 0 ? thr[0] : 0ull, nthr > 1 ? thr[1] : 0ull, nthr);
    return cudaGetLastError();
}

cudaError_t launch_check_packed(const uint64_t* p0, const uint64_t* p1, long long n, uint64_t valid,
                                unsigned int* err, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    long long nb = (n + 255) / 256;
    if (nb > 148 * 16) nb = 148 * 16;
    check_packed_kernel<<<(unsigned)nb, 256, 0, s>>>(p0, p1, n, valid, err);
    return cudaGetLastError();
}

__global__ void xor_into_kernel(uint64_t* dst, const uint64_t* src, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dst[i] ^= src[i];
}

cudaError_t launch_xor_rows(uint64_t* dst, const uint64_t* src, const uint64_t* /*unused*/, long long n,
                            cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    xor_into_kernel<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

// a few words device -> (mapped pinned host) memory by a kernel: no copy-engine transfer, so it does
// not queue behind a large download on the device-to-host engine
__global__ void copy_words_kernel(unsigned long long* dst, const unsigned long long* src, int n) {
    const int i = threadIdx.x;
    if (i < n) dst[i] = src[i];
}

// device-to-device copy of n u64 words by a kernel: the per-step row / plane copies stay off the copy
// engines, where they would queue behind an asynchronous lattice download
__global__ void copy_u64_kernel(uint64_t* __restrict__ dst, const uint64_t* __restrict__ src, long long n) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

cudaError_t launch_copy_u64(uint64_t* dst, const uint64_t* src, long long n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    long long nb = (n + 255) / 256;
    if (nb > 148 * 8) nb = 148 * 8;
    copy_u64_kernel<<<(unsigned)nb, 256, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

cudaError_t launch_copy_words(unsigned long long* dst, const unsigned long long* src, int n, cudaStream_t s) {
    if (n <= 0) return cudaSuccess;
    copy_words_kernel<<<1, 64, 0, s>>>(dst, src, n);
    return cudaGetLastError();
}

}  // namespace kmc
