// kmc_capi.cu -- host runtime and C ABI of libkmc_b200.so (declared in include/kmc.h).
//
// Owns: validation of the geometry (R6/R7), the rate table a1 (eq.(Arrhenius) P:963-968,
// Table COrates, R12-R14, quantised per R18), the schedule a2 (eq.(lie) P:395-401,
// eq.(strang), eq.(SLPCS); R1-R4, R20), the stream-ordered sub-step loop, the
// multi-GPU slab decomposition with its NCCL halo exchange a7 and the
// observables a8.  Product code; shares nothing with oracle/.
#include "kmc_internal.h"
#include "../../include/kmc.h"

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <dlfcn.h>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>

using namespace kmc;

#define KMC_VERSION "kmc_b200 0.1 (sm_100a)"

// ---------------------------------------------------------------------------------------------
// NCCL, loaded lazily with dlopen so the library loads on machines without it (world = 1).
// ---------------------------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    std::string err;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;
std::mutex g_nccl_mu;

bool load_nccl(std::string* why) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.tried) { if (!g_nccl.ok && why) *why = g_nccl.err; return g_nccl.ok; }
    g_nccl.tried = true;
    const char* env = getenv("KMC_NCCL_LIB");
    void* h = dlopen(env ? env : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) { g_nccl.err = std::string("dlopen libnccl.so.2 failed: ") + dlerror(); if (why) *why = g_nccl.err; return false; }
#define LOADSYM(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) { g_nccl.err = std::string("missing NCCL symbol ") + name; if (why) *why = g_nccl.err; return false; }
    LOADSYM(GetUniqueId, "ncclGetUniqueId");
    LOADSYM(CommInitRank, "ncclCommInitRank");
    LOADSYM(CommDestroy, "ncclCommDestroy");
    LOADSYM(Send, "ncclSend");
    LOADSYM(Recv, "ncclRecv");
    LOADSYM(GroupStart, "ncclGroupStart");
    LOADSYM(GroupEnd, "ncclGroupEnd");
    LOADSYM(AllReduce, "ncclAllReduce");
    LOADSYM(AllGather, "ncclAllGather");
    LOADSYM(GetErrorString, "ncclGetErrorString");
#undef LOADSYM
    g_nccl.ok = true;
    return true;
}

std::string g_create_error;

// Philox4x32-10 on the host (random schedule, R4).
void philox_host(uint32_t c[4], uint32_t k0, uint32_t k1) {
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c[0];
        const uint64_t p1 = (uint64_t)0xCD9E8D57u * c[2];
        const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c[1] ^ k0;
        const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c[3] ^ k1;
        c[1] = (uint32_t)p1;
        c[3] = (uint32_t)p0;
        c[0] = n0;
        c[2] = n2;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
}
}  // namespace

struct VgShared {
    cudaStream_t stream = nullptr;
    int refs = 0;
};

struct kmc_ctx {
    kmc_geometry geom{};
    kmc_model model{};
    int rank = 0, world = 1, device = 0;
    int kind = 0, nplanes = 1, nstates = 2, C = 2;
    bool cross = false;             // events write outside the anchor cell
    Geo g{};
    long long H_local = 0, W = 0;
    // rate table
    int nclass = 0, F = 0;
    int ctype[kMaxClass], cdir[kMaxClass], ckappa[kMaxClass];
    double crate[kMaxClass];
    uint64_t crate_u64[kMaxClass];
    // device state
    uint64_t* planes[2] = {nullptr, nullptr};
    long long plane_words = 0;
    uint32_t* wev = nullptr;
    uint32_t* wmark = nullptr;               // f4: per-cell counters at the last kmc_workload_mark
    bool fused = false;                      // fused halo exchange (peer writes inside the window kernel)
    bool borrowed = false;                   // planes are the caller's buffer (kmc_attach_planes)
    bool fused_ipc = false;                  // ... across GPUs: CUDA-IPC peer planes + device flags
    unsigned long long* flags = nullptr;     // [2]: written by the up / down neighbour
    unsigned long long* peer_up_flags = nullptr;
    unsigned long long* peer_dn_flags = nullptr;
    unsigned long long epoch = 0;            // fused windows completed
    std::vector<void*> ipc_open;             // IPC mappings to close at destroy
    uint64_t* peer_up[2] = {nullptr, nullptr};
    uint64_t* peer_dn[2] = {nullptr, nullptr};
    int peer_up_rows = 0;
    unsigned long long* strips = nullptr;    // f4: strip loads [M strips] + inclusive cdf [M]
    long long strips_n = 0;
    long long* wl_out = nullptr;             // f4: device bounds [P+1] + 2 doubles (imbalance)
    unsigned long long* ev_total = nullptr;
    unsigned long long* series = nullptr;    // f1 coverage process: [series_cap][R local] counts (R30)
    long long series_cap = 0, series_n = 0;
    int series_state = 1;
    unsigned int* queue = nullptr;           // window kernel's dynamic chunk counter
    unsigned long long* obs_buf = nullptr;   // KMC_OBS_WORDS (enqueue_obs layout)
    unsigned long long* obs_acc = nullptr;   // kObsCounters + 1: the observables kernel's accumulator + ticket
    double2* logtab = nullptr;               // log_spec table {c_j, L_j}
    unsigned int* err_flag = nullptr;
    uint8_t* staging = nullptr;              // uint8 local slab (set/get_config from host)
    uint64_t* ghost_snap = nullptr;          // [2 rows][nplanes] snapshot / delta buffers (world > 1)
    uint64_t* ghost_recv = nullptr;
    unsigned long long* h_obs = nullptr;     // pinned, mapped: the observables kernel writes it directly
    unsigned long long* d_hobs = nullptr;    // device alias of h_obs (no copy engine: a pending download
                                             // on the copy stream does not delay kmc_observables)
    unsigned long long* h_flag = nullptr;    // pinned: fused-exchange timeout word (world > 1)
    unsigned int* h_err = nullptr;           // pinned (set_config validation flag)
    uint64_t* spare[2] = {nullptr, nullptr}; // set_config double buffer
    uint64_t* spare2[2] = {nullptr, nullptr};// third buffer: a staged upload while the previous planes download
    // pipelined upload (kmc_stage_config_packed / kmc_commit_config): H2D + validation of the next
    // configuration into the spare planes on a copy stream, overlapping the windows in flight
    cudaStream_t copy_stream = nullptr;      // H2D of staged uploads
    cudaStream_t dl_stream = nullptr;        // D2H of kmc_download_config_packed (own stream: the PCIe
                                             // link is full duplex, so a download overlaps the next upload)
    cudaEvent_t staged_ev = nullptr;         // copy + check of the staged configuration done
    cudaEvent_t consumed_ev = nullptr;       // every window that read the current spare has been enqueued before it
    bool staged = false, consumed_valid = false;
    unsigned int* stage_err = nullptr;       // device alias of h_stage_err (mapped pinned memory)
    unsigned int* h_stage_err = nullptr;     // pinned, mapped: the staged check writes it directly (no
                                             // D2H copy, which would queue behind a pending download
                                             // on the device-to-host copy engine)
    // asynchronous download (kmc_download_config_packed): D2H of the planes on the copy stream; a
    // stream-ordered guard keeps the downloaded buffers unchanged until the copy has finished
    cudaEvent_t dl_ev = nullptr, dl_start_ev = nullptr;
    bool dl_pending = false;
    const uint64_t* dl_buf = nullptr;        // planes[0] at download time (the buffer pair being read)
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    bool vgroup = false;                     // virtual rank of a kmc_vgroup_create group (no NCCL)
    double rate_per_cell = 0.0;            // rough events per unit time per cell (kernel choice)
    int kernel_mode = 0;                     // kmc_set_kernel
    SubstepArgs args{};                      // window-invariant kernel arguments (build_args_template)
    struct VgShared* vg_shared = nullptr;    // virtual-rank group stream (reference counted)
    // schedule state
    uint64_t window = 0;
    double time = 0.0;
    // timing
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> tev;
    size_t tev_used = 0;
    // multi-GPU
    ncclComm_t comm = nullptr;
    int rank_up = -1, rank_down = -1;        // -y and +y ring neighbours (2D slabs)
    std::vector<int64_t> bounds;             // 2D: cell-row bounds of every rank's slab (world + 1)
    std::string err;
};

namespace {

kmc_status fail(kmc_ctx* c, kmc_status s, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf; else g_create_error = buf;
    return s;
}

#define CUDA_TRY(ctx, call) do { cudaError_t e_ = (call); if (e_ != cudaSuccess) \
    return fail(ctx, KMC_ECUDA, "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); } while (0)
#define NCCL_TRY(ctx, call) do { ncclResult_t r_ = (call); if (r_ != ncclSuccess) \
    return fail(ctx, KMC_ENCCL, "%s: %s", #call, g_nccl.GetErrorString ? g_nccl.GetErrorString(r_) : "?"); } while (0)

int types_per_site(int kind, int z) {
    switch (kind) {
    case KMC_ADSDES: return 2;
    case KMC_ADSDES_DIFF: return 2 + z;
    case KMC_ZGB: return 1 + 3 * z;
    case KMC_ZGB_DIFF: return 1 + 4 * z;
    case KMC_ZGB_ODIFF: return 1 + 4 * z;
    }
    return 0;
}

// a1: class list in canonical order with FP64 rates.
int build_classes(const kmc_model& m, int ndim, int* type, int* dir, int* kappa, double* rate) {
    const int z = 2 * ndim;
    int n = 0;
    auto add = [&](int t, int d, int k, double r) { type[n] = t; dir[n] = d; kappa[n] = k; rate[n] = r; ++n; };
    if (m.kind == KMC_ADSDES || m.kind == KMC_ADSDES_DIFF) {
        add(T_ADS, -1, 0, m.ca);                                   // c1 (1 - sigma)
        for (int nn = 0; nn <= z; ++nn) {                          // c2 sigma exp(-beta U), U = K n + h
            double u = m.K * (double)nn;
            u = u + m.h;
            u = m.beta * u;
            u = -u;
            add(T_DES, -1, nn, m.cd * std::exp(u));
        }
        if (m.kind == KMC_ADSDES_DIFF)
            for (int nn = 0; nn < z; ++nn)                         // R31: n-major, direction inner
                for (int d = 0; d < z; ++d) {                      // R12: c_hop exp(-beta K n(x))
                    double u = m.K * (double)nn;
                    u = m.beta * u;
                    u = -u;
                    add(T_HOP, d, nn, m.c_hop * std::exp(u));
                }
        return n;
    }
    add(T_COADS, -1, 0, m.k1);
    for (int d = 0; d < z; ++d) add(T_O2ADS, d, 0, (1.0 - m.k1) / (double)z);
    for (int d = 0; d < z; ++d) add(T_RCO, d, 0, m.k2 / (double)z);
    for (int d = 0; d < z; ++d) add(T_RO, d, 0, m.k2 / (double)z);
    if (m.kind == KMC_ZGB_DIFF)
        for (int d = 0; d < z; ++d) add(T_COHOP, d, 0, m.c_hop);
    if (m.kind == KMC_ZGB_ODIFF)   // fast O diffusion (R33): O(x), vacant x+e_d -> vacant, O
        for (int d = 0; d < z; ++d) add(T_OHOP, d, 0, m.c_hop);
    return n;
}

// R18 quantisation; returns F or -1.
int quantise(const double* rate, int n, long long slots_bound, uint64_t* out) {
    double rmax = 0.0;
    for (int i = 0; i < n; ++i) {
        if (!(rate[i] >= 0.0) || std::isinf(rate[i])) return -1;
        rmax = rate[i] > rmax ? rate[i] : rmax;
    }
    int F = 0;
    if (rmax > 0.0) {
        int e = 0;
        const double mant = std::frexp(rmax * (double)slots_bound, &e);
        const int ceil_log2 = (mant == 0.5) ? e - 1 : e;
        F = 62 - ceil_log2;
        if (F < 0) return -1;
    }
    for (int i = 0; i < n; ++i) out[i] = (uint64_t)std::llround(std::ldexp(rate[i], F));
    return F;
}

uint64_t lowmask(int nbits) { return nbits >= 64 ? ~0ull : ((1ull << nbits) - 1ull); }

long long active_cells(const kmc_ctx* c) {
    const long long half = c->g.Mx / 2;
    if (c->g.ndim == 1) return half * c->g.R;
    const long long rows = (c->C == 2) ? c->g.My_local : c->g.My_local / 2;
    return half * c->g.R * rows;
}

// a7 forward exchange (world > 1, 2D): owned boundary cell rows -> neighbours' ghost rows.
// f1 (R30): append one sample of the coverage process (per-replica count of series_state over the
// owned cells) to the device series; stream-ordered, no host synchronisation.  Full: no-op.
kmc_status fused_quiesce(kmc_ctx* c);

kmc_status record_sample(kmc_ctx* c) {
    if (!c->series || c->series_n >= c->series_cap) return KMC_OK;
    kmc_status sq = fused_quiesce(c);
    if (sq != KMC_OK) return sq;
    unsigned long long* out = c->series + (size_t)c->series_n * c->g.R;
    CUDA_TRY(c, cudaMemsetAsync(out, 0, (size_t)c->g.R * 8, c->stream));
    SeriesArgs a{};
    a.g = c->g;
    a.plane0 = c->planes[0];
    a.plane1 = c->planes[1];
    a.nplanes = c->nplanes;
    a.state = c->series_state;
    a.out = out;
    CUDA_TRY(c, launch_series_count(a, c->stream));
    ++c->series_n;
    return KMC_OK;
}

// A pending asynchronous download reads the buffer pair whose plane 0 is dl_buf: before work on the
// context's stream overwrites that pair (windows, exchanges, uploads), the stream waits for the copy.
// A committed staged configuration swaps other buffers in, so the windows after it never wait.
kmc_status dl_guard(kmc_ctx* c, const uint64_t* target) {
    if (c->dl_pending && target == c->dl_buf) {
        CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->dl_ev, 0));
        c->dl_pending = false;               // everything later on the stream is ordered after the copy
    }
    return KMC_OK;
}

kmc_status exchange_forward(kmc_ctx* c) {
    if (!c->comm || !c->g.ghost) return KMC_OK;   // world 1 (no ring), 1D, vgroup (exchanged by its driver)
    kmc_status sg = dl_guard(c, c->planes[0]);
    if (sg != KMC_OK) return sg;
    const size_t rowlen = (size_t)c->g.R * c->g.Mx;
    const int My = c->g.My_local;
    NCCL_TRY(c, g_nccl.GroupStart());
    for (int p = 0; p < c->nplanes; ++p) {
        uint64_t* pl = c->planes[p];
        // order matters when rank_up == rank_down (world = 2): last row first, then first row
        NCCL_TRY(c, g_nccl.Send(pl + (size_t)My * rowlen, rowlen * 8, ncclUint8, c->rank_down, c->comm, c->stream));
        NCCL_TRY(c, g_nccl.Send(pl + rowlen, rowlen * 8, ncclUint8, c->rank_up, c->comm, c->stream));
        NCCL_TRY(c, g_nccl.Recv(pl, rowlen * 8, ncclUint8, c->rank_up, c->comm, c->stream));
        NCCL_TRY(c, g_nccl.Recv(pl + (size_t)(My + 1) * rowlen, rowlen * 8, ncclUint8, c->rank_down, c->comm, c->stream));
    }
    NCCL_TRY(c, g_nccl.GroupEnd());
    if (c->cross) {   // snapshot the ghost rows so the sub-step's writes into them can be sent back
        for (int p = 0; p < c->nplanes; ++p) {
            CUDA_TRY(c, launch_copy_u64(c->ghost_snap + (size_t)(2 * p) * rowlen, c->planes[p], (long long)rowlen, c->stream));
            CUDA_TRY(c, launch_copy_u64(c->ghost_snap + (size_t)(2 * p + 1) * rowlen, c->planes[p] + (size_t)(My + 1) * rowlen,
                                        (long long)rowlen, c->stream));
        }
    }
    return KMC_OK;
}

// a7 reverse exchange for cross-cell-writing models: ghost-row deltas back to their owners,
// merged by XOR (same-colour closures are disjoint, R6, so exactly one writer per bit).
kmc_status exchange_reverse(kmc_ctx* c) {
    if (!c->comm || !c->g.ghost || !c->cross) return KMC_OK;
    kmc_status sg = dl_guard(c, c->planes[0]);
    if (sg != KMC_OK) return sg;
    const size_t rowlen = (size_t)c->g.R * c->g.Mx;
    const int My = c->g.My_local;
    for (int p = 0; p < c->nplanes; ++p) {   // snap := ghost XOR snap  (the delta)
        CUDA_TRY(c, launch_xor_rows(c->ghost_snap + (size_t)(2 * p) * rowlen, c->planes[p], nullptr, (long long)rowlen, c->stream));
        CUDA_TRY(c, launch_xor_rows(c->ghost_snap + (size_t)(2 * p + 1) * rowlen, c->planes[p] + (size_t)(My + 1) * rowlen,
                                    nullptr, (long long)rowlen, c->stream));
    }
    NCCL_TRY(c, g_nccl.GroupStart());
    for (int p = 0; p < c->nplanes; ++p) {
        // send: top-ghost delta -> up (its last row), bottom-ghost delta -> down (its first row)
        NCCL_TRY(c, g_nccl.Send(c->ghost_snap + (size_t)(2 * p) * rowlen, rowlen * 8, ncclUint8, c->rank_up, c->comm, c->stream));
        NCCL_TRY(c, g_nccl.Send(c->ghost_snap + (size_t)(2 * p + 1) * rowlen, rowlen * 8, ncclUint8, c->rank_down, c->comm, c->stream));
        // receive (same per-peer order as the peer's sends): delta for my last row from down, first row from up
        NCCL_TRY(c, g_nccl.Recv(c->ghost_recv + (size_t)(2 * p + 1) * rowlen, rowlen * 8, ncclUint8, c->rank_down, c->comm, c->stream));
        NCCL_TRY(c, g_nccl.Recv(c->ghost_recv + (size_t)(2 * p) * rowlen, rowlen * 8, ncclUint8, c->rank_up, c->comm, c->stream));
    }
    NCCL_TRY(c, g_nccl.GroupEnd());
    for (int p = 0; p < c->nplanes; ++p) {
        CUDA_TRY(c, launch_xor_rows(c->planes[p] + rowlen, c->ghost_recv + (size_t)(2 * p) * rowlen, nullptr,
                                    (long long)rowlen, c->stream));
        CUDA_TRY(c, launch_xor_rows(c->planes[p] + (size_t)My * rowlen, c->ghost_recv + (size_t)(2 * p + 1) * rowlen,
                                    nullptr, (long long)rowlen, c->stream));
    }
    return KMC_OK;
}

// One window's kernel (a3-a6) on this rank's owned cells of `colour`; advances the window counter.
// class_mask: bit i set = class i active in this window (multiscale sub-steps, f2); the rates of
// inactive classes are 0, so they never fire and add nothing to lambda.
// The window-invariant kernel arguments (geometry, keys, Philox round keys, rate table, log
// tables), built once at create so a window launch only fills in colour, duration and window id.
void build_args_template(kmc_ctx* c) {
    SubstepArgs& a = c->args;
    a = SubstepArgs{};
    a.g = c->g;
    a.wev = c->wev;
    a.ev_total = c->ev_total;
    a.queue = c->queue;
    a.C = c->C;
    a.inv_scale = std::ldexp(1.0, -c->F);
    a.refill_min = 1;                       // set per window (launch_window)
    a.half = (uint32_t)(c->g.Mx / 2);
    a.inv_half = 1.0 / (double)a.half;
    a.inv_R = 1.0 / (double)c->g.R;
    a.key0 = (uint32_t)c->geom.seed;
    a.key1 = (uint32_t)(c->geom.seed >> 32);
    for (int i = 0; i < 10; ++i) {
        a.rk0[i] = a.key0 + (uint32_t)i * 0x9E3779B9u;
        a.rk1[i] = a.key1 + (uint32_t)i * 0xBB67AE85u;
    }
    for (int i = 0; i < c->nclass; ++i) a.rate[i] = c->crate_u64[i];
    a.logtab = c->logtab;
    a.lcoef[0] = 0x1.2492492492492p-3;      // 1/7
    a.lcoef[1] = -0x1.5555555555555p-3;     // -1/6
    a.lcoef[2] = 0x1.999999999999ap-3;      // 1/5
    a.lcoef[3] = 0x1.5555555555555p-2;      // 1/3
    a.lcoef[4] = 0x1.62e42feep-1;           // ln2_hi (fdlibm)
    a.lcoef[5] = 0x1.a39ef35793c76p-33;     // ln2_lo (fdlibm)
}

// f3 nested decomposition (R28): restrict a window to the outer blocks of one outer colour.
struct Nest {
    int outer;    // outer colour 0/1
    int block;    // outer block size in cell rows (2D) or cells (1D)
};

// Fills the nested fields of the kernel arguments; returns the number of active cells.
long long apply_nest(const kmc_ctx* c, const Nest& n, SubstepArgs& a) {
    const long long half = c->g.Mx / 2;
    a.nest = 1;
    a.nest_B = n.block;
    if (c->g.ndim == 1) {              // blocks of B cells along x; B/2 colour pairs per block
        const long long nblk = c->g.Mx / n.block;
        a.nest_s = n.outer;
        a.nest_rows = (uint32_t)(n.block / 2);
        a.half = (uint32_t)((nblk / 2) * (n.block / 2));
        a.inv_half = 1.0 / (double)a.half;
        a.inv_nest_rows = 1.0 / (double)a.nest_rows;
        return (long long)a.half * c->g.R;
    }
    const int nblk_loc = c->g.My_local / n.block;
    a.nest_s = (n.outer + c->g.row_offset / n.block) & 1;   // local block 0 is global block row_offset/B
    const int n_o = (nblk_loc - a.nest_s + 1) / 2;           // local blocks of this outer colour
    a.nest_rows = (uint32_t)(c->C == 2 ? n.block : n.block / 2);
    a.inv_nest_rows = 1.0 / (double)a.nest_rows;
    return half * c->g.R * (long long)n_o * a.nest_rows;
}

// The kernel arguments of window c->window + ahead (colour, duration D; class_mask: multiscale rate
// subset; nest: f3 outer blocks) and its number of active cells.
static SubstepArgs window_args(const kmc_ctx* c, int colour, double D, uint64_t class_mask, const Nest* nest,
                               uint64_t ahead, long long* nactive_out) {
    SubstepArgs a = c->args;
    a.plane0 = c->planes[0];                // (set_config swaps plane buffers)
    a.plane1 = c->planes[1];
    a.colour = colour;
    a.D = D;
    *nactive_out = nest ? apply_nest(c, *nest, a) : active_cells(c);
    if (c->fused && !nest) {
        for (int p = 0; p < 2; ++p) { a.peer_up[p] = c->peer_up[p]; a.peer_dn[p] = c->peer_dn[p]; }
        a.peer_up_rows = c->peer_up_rows;
    }
    // refill batching of the window kernel (performance only; results are bit-identical): a warp
    // refills its finished lanes once refill_min of them are parked.  Best thresholds measured on
    // B200 (KMC_REFILL sweeps) fall with the events per cell-window mu: mu >= 16 (D x rate_per_cell,
    // Ising dt = 1, diffusion dt = 1): spin flip 3, diffusion 4; below (dt = 0.01, ZGB at dt = 0.1):
    // spin flip 10 (flat from 2 to 12 at mu ~ 0.8), diffusion 10, ZGB 14 (mu ~ 2.3; 2.105e10 vs 1.94e10
    // at 8), ZGB + CO hops 10 (mu ~ 4.3; +4 % over 16), ZGB + O hops 8 (mu ~ 6.5; +10 % over 16).
    // Env KMC_REFILL overrides.
    static const int refill_env = [] { const char* e = getenv("KMC_REFILL"); return e ? atoi(e) : 0; }();
    static const int refill_hi[5] = {3, 4, 6, 6, 6}, refill_lo[5] = {10, 10, 14, 10, 8};   // by model kind
    a.refill_min = refill_env >= 1 && refill_env <= 32 ? refill_env
                 : (D * c->rate_per_cell >= 16.0 ? refill_hi[c->kind] : refill_lo[c->kind]);
    const uint64_t w = c->window + ahead;
    a.w_lo = (uint32_t)w;
    a.w_hi_tag = (uint32_t)((w >> 32) & 0x0FFFFFFFu);   // tag EVT = 0 (R17)
    if (class_mask != ~0ull)
        for (int i = 0; i < c->nclass; ++i) a.rate[i] = ((class_mask >> i) & 1ull) ? c->crate_u64[i] : 0ull;
    if (c->kind == KMC_ADSDES_DIFF) {   // R31 hop blocks: one rate per block -> the block-walk kernel
        const int z = 2 * c->g.ndim;
        a.hop_fast = 1;
        for (int n = 0; n < z; ++n) {
            const uint64_t r = a.rate[2 + z + n * z];
            for (int d = 1; d < z; ++d) a.hop_fast &= a.rate[2 + z + n * z + d] == r ? 1 : 0;
            a.hopz[n] = (uint64_t)(z - n) * r;
        }
        static const int hop_env = [] { const char* e = getenv("KMC_HOPFAST"); return e ? atoi(e) : 1; }();
        if (!hop_env) a.hop_fast = 0;
    } else if (c->kind >= KMC_ZGB) {   // ZGB*: one rate per direction group
        const int z = 2 * c->g.ndim;
        a.hop_fast = 1;
        for (int i = 1; i < c->nclass; ++i)
            a.hop_fast &= a.rate[i] == a.rate[1 + ((i - 1) / z) * z] ? 1 : 0;
    }
    // lanes per cell (spin flip): 0 = auto (group_size), 1 = the queue kernel, g = forced groups
    const int mode = c->kernel_mode;
    a.group = mode == KMC_KERNEL_QUEUE ? 1 : mode >= KMC_KERNEL_GROUP2 ? (1 << (mode - KMC_KERNEL_GROUP2 + 1)) : 0;
    return a;
}

// kernel timing (kmc_enable_timing): an event pair around a launch
static kmc_status timing_begin(kmc_ctx* c, cudaEvent_t* e1) {
    *e1 = nullptr;
    if (!c->timing) return KMC_OK;
    if (c->tev_used == c->tev.size()) {
        cudaEvent_t x, y;
        CUDA_TRY(c, cudaEventCreate(&x));
        CUDA_TRY(c, cudaEventCreate(&y));
        c->tev.emplace_back(x, y);
    }
    *e1 = c->tev[c->tev_used].second;
    CUDA_TRY(c, cudaEventRecord(c->tev[c->tev_used].first, c->stream));
    ++c->tev_used;
    return KMC_OK;
}

kmc_status launch_window(kmc_ctx* c, int colour, double D, uint64_t class_mask = ~0ull, const Nest* nest = nullptr) {
    kmc_status sg = dl_guard(c, c->planes[0]);
    if (sg != KMC_OK) return sg;
    long long nactive = 0;
    SubstepArgs a = window_args(c, colour, D, class_mask, nest, 0, &nactive);
    cudaEvent_t e1 = nullptr;
    kmc_status st = timing_begin(c, &e1);
    if (st != KMC_OK) return st;
    // kernel choice: the shared-memory tile kernel for 2D spin-flip windows (KMC_TILE=0 forces the
    // lane-queue kernel, KMC_TILE=1 the tile kernel); both give bit-identical results
    static const int tile_env = [] { const char* e = getenv("KMC_TILE"); return e ? atoi(e) : -1; }();
    int mode = c->kernel_mode;                                   // kmc_set_kernel: 0 auto, 1 queue, 2 tile, 3.. groups
    if (mode == KMC_KERNEL_AUTO && tile_env >= 0) mode = tile_env ? KMC_KERNEL_TILE : KMC_KERNEL_QUEUE;
    // auto never picks the tile kernel: measured on B200 it is 4-17 % slower at dt = 1 and dt = 0.01
    // (both regimes are instruction-issue bound, not load-latency bound); it stays selectable
    const bool use_tile = c->kind == KMC_ADSDES && c->g.ndim == 2 && mode == KMC_KERNEL_TILE && !nest;
    cudaError_t le = use_tile ? launch_substep_tile(a, c->stream) : cudaErrorNotSupported;
    if (le == cudaSuccess && use_tile) le = queue_slot_reset(a, c->stream);
    if (le == cudaErrorNotSupported) le = launch_substep(c->kind, a, nactive, c->stream);
    CUDA_TRY(c, le);
    if (e1) CUDA_TRY(c, cudaEventRecord(e1, c->stream));
    c->window += 1;
    return KMC_OK;
}

// Fused exchange across GPUs: the neighbours' windows write into this rank's boundary and ghost rows
// through peer memory, so ANY other use of the planes (exchange, upload, download, observables,
// coverage samples, random init) is first ordered after both neighbours' last window: a one-thread
// wait kernel on the device flags, stream-ordered (no host synchronisation).
kmc_status fused_quiesce(kmc_ctx* c) {
    if (c->fused_ipc) CUDA_TRY(c, launch_wait_flags(c->flags, c->epoch, c->stream));
    return KMC_OK;
}

// ... and the ghost rows are refreshed by one NCCL exchange at the start of every call that runs
// windows (configuration uploads may have changed the neighbours' rows); afterwards the window
// kernels keep them current.  Every rank makes the same calls, so this stays collective.
kmc_status fused_refresh(kmc_ctx* c) {
    if (!c->fused_ipc) return KMC_OK;
    kmc_status st = fused_quiesce(c);
    return st != KMC_OK ? st : exchange_forward(c);
}

kmc_status do_substep(kmc_ctx* c, int colour, double D, uint64_t class_mask = ~0ull) {
    if (colour < 0 || colour >= c->C) return fail(c, KMC_EINVAL, "colour %d out of range [0,%d)", colour, c->C);
    if (!(D >= 0.0)) return fail(c, KMC_EINVAL, "window duration must be >= 0");
    if (c->fused_ipc) {
        // fused exchange across GPUs: wait for both neighbours' previous window, run the window
        // (its kernel writes the neighbours' shared rows through NVLink), signal completion
        CUDA_TRY(c, launch_wait_flags(c->flags, c->epoch, c->stream));
        kmc_status st = launch_window(c, colour, D, class_mask);
        if (st != KMC_OK) return st;
        ++c->epoch;
        CUDA_TRY(c, launch_signal_flags(c->peer_up_flags, c->peer_dn_flags, c->epoch, c->stream));
        return KMC_OK;
    }
    kmc_status st = exchange_forward(c);
    if (st != KMC_OK) return st;
    st = launch_window(c, colour, D, class_mask);
    if (st != KMC_OK) return st;
    return exchange_reverse(c);
}

int random_colour(uint64_t seed, uint64_t w, int C) {
    uint32_t ctr[4] = {0u, 0u, (uint32_t)w, (uint32_t)((w >> 32) & 0x0FFFFFFFu) | (1u << 28)};   // tag SCHED
    philox_host(ctr, (uint32_t)seed, (uint32_t)(seed >> 32));
    return (int)(((uint64_t)C * ctr[0]) >> 32);
}

// a2: the sub-steps (colour, duration) of one macro-step of duration d starting at window w0.
std::vector<std::pair<int, double>> macro_schedule(int scheme, int C, double d, uint64_t seed, uint64_t w0) {
    std::vector<std::pair<int, double>> s;
    const double h = d * 0.5;
    if (scheme == KMC_LIE) {                        // eq.(lie), colour 0 first (R1)
        for (int col = 0; col < C; ++col) s.emplace_back(col, d);
    } else if (scheme == KMC_STRANG) {              // eq.(strang), halves to colour 0 (R2)
        if (C == 2) s = {{0, h}, {1, d}, {0, h}};
        else s = {{0, h}, {1, h}, {2, h}, {3, d}, {2, h}, {1, h}, {0, h}};
    } else {                                        // eq.(SLPCS): C windows, xi_w by window id (R4)
        for (int k = 0; k < C; ++k) s.emplace_back(random_colour(seed, w0 + (uint64_t)k, C), d);
    }
    return s;
}

// R20: macro-step durations of kmc_run(T, dt).
std::vector<double> macro_durations(double T, double dt, bool* truncated) {
    std::vector<double> out;
    *truncated = false;
    if (T == 0.0) return out;
    long long n = (long long)std::ceil(T / dt - 1e-9);
    if (n < 1) n = 1;
    double last = T - (double)(n - 1) * dt;
    *truncated = true;
    if (std::fabs(last - dt) <= 1e-9 * dt) { last = dt; *truncated = false; }
    out.assign((size_t)n, dt);
    out.back() = last;
    return out;
}

// f3 (R28): validation of a nested run and its outer factor list for one macro-step d.
kmc_status check_nested(kmc_ctx* c, double T, double dt, int n_inner, int outer, int inner, int block) {
    if (!(dt > 0.0) || !(T >= 0.0) || std::isinf(T)) return fail(c, KMC_EINVAL, "need dt > 0 and finite T >= 0");
    if (outer != KMC_LIE && outer != KMC_STRANG) return fail(c, KMC_EINVAL, "nested outer scheme must be Lie or Strang");
    if (inner < KMC_LIE || inner > KMC_RANDOM) return fail(c, KMC_EINVAL, "unknown inner scheme %d", inner);
    if (n_inner < 1) return fail(c, KMC_EINVAL, "n_inner must be >= 1");
    if (block < 2 || block % 2) return fail(c, KMC_EINVAL, "nested block must be even and >= 2");
    if (c->g.ndim == 1) {
        if (c->g.Mx % (2 * block)) return fail(c, KMC_EPARTITION, "nested: %d cells not a multiple of 2*block", c->g.Mx);
    } else {
        // the GLOBAL cell-row count (uneven slabs: not My_local x world), so every rank agrees
        const long long rows = c->geom.dims[0] / c->g.qy;
        if (rows % (2 * block)) return fail(c, KMC_EPARTITION, "nested: %lld cell rows not a multiple of 2*block", rows);
        // outer blocks must not straddle ranks: then a rank's ghost rows belong to the other outer
        // colour for a whole outer factor, and one exchange per outer factor suffices.  Checked on
        // EVERY slab bound (all ranks hold the same bounds), so no rank enters the collective
        // exchange while another one fails here.
        if (c->world > 1)
            for (size_t r = 0; r < c->bounds.size(); ++r)
                if (c->bounds[r] % block)
                    return fail(c, KMC_EPARTITION, "nested: slab bound %lld (cell rows) not a multiple of block",
                                (long long)c->bounds[r]);
    }
    return KMC_OK;
}

std::vector<std::pair<int, double>> outer_factors(int outer, double d) {
    if (outer == KMC_LIE) return {{0, d}, {1, d}};
    return {{0, d * 0.5}, {1, d}, {0, d * 0.5}};
}

// ---- virtual ranks: G slabs of one lattice on one device, exchanged by stream-ordered copies ----
// Same partition and exchange protocol as the NCCL path (exchange_forward / exchange_reverse), run
// in lockstep by one host thread, so the multi-rank logic can be checked on a single GPU.
kmc_status vgroup_forward(kmc_ctx** cs, int world) {
    for (int r = 0; r < world; ++r) {
        kmc_ctx* c = cs[r];
        const size_t rowlen = (size_t)c->g.R * c->g.Mx;
        const int My = c->g.My_local;
        kmc_ctx* up = cs[c->rank_up];
        kmc_ctx* dn = cs[c->rank_down];
        for (int p = 0; p < c->nplanes; ++p) {
            CUDA_TRY(c, cudaMemcpyAsync(c->planes[p], up->planes[p] + (size_t)up->g.My_local * rowlen, rowlen * 8,
                                        cudaMemcpyDeviceToDevice, c->stream));
            CUDA_TRY(c, cudaMemcpyAsync(c->planes[p] + (size_t)(My + 1) * rowlen, dn->planes[p] + rowlen, rowlen * 8,
                                        cudaMemcpyDeviceToDevice, c->stream));
            if (c->cross) {
                CUDA_TRY(c, cudaMemcpyAsync(c->ghost_snap + (size_t)(2 * p) * rowlen, c->planes[p], rowlen * 8,
                                            cudaMemcpyDeviceToDevice, c->stream));
                CUDA_TRY(c, cudaMemcpyAsync(c->ghost_snap + (size_t)(2 * p + 1) * rowlen, c->planes[p] + (size_t)(My + 1) * rowlen,
                                            rowlen * 8, cudaMemcpyDeviceToDevice, c->stream));
            }
        }
    }
    return KMC_OK;
}

kmc_status vgroup_reverse(kmc_ctx** cs, int world) {
    for (int r = 0; r < world; ++r) {
        kmc_ctx* c = cs[r];
        if (!c->cross) return KMC_OK;
        const size_t rowlen = (size_t)c->g.R * c->g.Mx;
        const int My = c->g.My_local;
        kmc_ctx* up = cs[c->rank_up];
        kmc_ctx* dn = cs[c->rank_down];
        for (int p = 0; p < c->nplanes; ++p) {
            uint64_t* dtop = c->ghost_snap + (size_t)(2 * p) * rowlen;
            uint64_t* dbot = c->ghost_snap + (size_t)(2 * p + 1) * rowlen;
            CUDA_TRY(c, launch_xor_rows(dtop, c->planes[p], nullptr, (long long)rowlen, c->stream));
            CUDA_TRY(c, launch_xor_rows(dbot, c->planes[p] + (size_t)(My + 1) * rowlen, nullptr, (long long)rowlen, c->stream));
            CUDA_TRY(c, launch_xor_rows(up->planes[p] + (size_t)up->g.My_local * rowlen, dtop, nullptr, (long long)rowlen, c->stream));
            CUDA_TRY(c, launch_xor_rows(dn->planes[p] + rowlen, dbot, nullptr, (long long)rowlen, c->stream));
        }
    }
    return KMC_OK;
}

}  // namespace

// ---------------------------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------------------------
static kmc_status create_ctx(const kmc_geometry* geom, const kmc_model* model, const kmc_dist* dist, bool vgroup,
                             kmc_ctx** out);

extern "C" {

const char* kmc_version(void) { return KMC_VERSION; }

void kmc_abi_sizes(int64_t out[4]) {
    if (!out) return;
    out[0] = (int64_t)sizeof(kmc_geometry);
    out[1] = (int64_t)sizeof(kmc_model);
    out[2] = (int64_t)sizeof(kmc_dist);
    out[3] = (int64_t)sizeof(kmc_obs);
}
const char* kmc_create_error(void) { return g_create_error.c_str(); }
const char* kmc_last_error(const kmc_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

kmc_status kmc_partition_plan(const kmc_geometry* geom, int32_t kind, int32_t world, int32_t rank, int64_t out[6]) {
    if (!geom || !out || world < 1 || rank < 0 || rank >= world) return fail(nullptr, KMC_EINVAL, "bad partition arguments");
    const bool cross = kind != KMC_ADSDES;
    if (geom->ndim == 1) {
        if (geom->replicas % world) return fail(nullptr, KMC_EPARTITION, "1D: replicas %d not divisible by world %d", geom->replicas, world);
        const int64_t rl = geom->replicas / world;
        out[0] = rank * rl; out[1] = rl; out[2] = 0; out[3] = 1; out[4] = -1; out[5] = -1;
        return KMC_OK;
    }
    const int64_t H = geom->dims[0];
    const int qy = geom->cell[0];
    if (qy <= 0 || H % ((int64_t)world * 2 * qy))
        return fail(nullptr, KMC_EPARTITION, "2D: rows %lld not a multiple of world*2*q_y = %lld", (long long)H,
                    (long long)world * 2 * qy);
    const int64_t rows_cells = H / qy / world;
    out[0] = 0; out[1] = geom->replicas; out[2] = rank * rows_cells; out[3] = rows_cells;
    out[4] = world > 1 ? (rank + world - 1) % world : -1;
    out[5] = world > 1 ? (rank + 1) % world : -1;
    (void)cross;
    return KMC_OK;
}

kmc_status kmc_nccl_unique_id(uint8_t out[128]) {
    std::string why;
    if (!out) return fail(nullptr, KMC_EINVAL, "NULL out");
    if (!load_nccl(&why)) return fail(nullptr, KMC_ENCCL, "%s", why.c_str());
    ncclUniqueId id;
    ncclResult_t r = g_nccl.GetUniqueId(&id);
    if (r != ncclSuccess) return fail(nullptr, KMC_ENCCL, "ncclGetUniqueId: %s", g_nccl.GetErrorString(r));
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    memcpy(out, &id, 128);
    return KMC_OK;
}

kmc_status kmc_create(const kmc_geometry* geom, const kmc_model* model, const kmc_dist* dist, kmc_ctx** out) {
    return create_ctx(geom, model, dist, false, out);
}

}  // extern "C"

// Fused exchange across GPUs (kmc_dist.fused_exchange): every rank exports its plane buffers and a
// 2-word flag array as CUDA-IPC handles; an NCCL all-gather gives every rank its ring neighbours'
// handles and slab heights; the neighbours' planes and flags are mapped into this process (NVLink
// peer memory).  The window kernel then writes the shared rows directly (PEER variant) and
// do_substep orders windows with the device flags instead of NCCL send/recv.
static bool setup_fused_ipc(kmc_ctx* c, std::string* why) {
    struct Blob { cudaIpcMemHandle_t planes[2]; cudaIpcMemHandle_t flags; long long rows; };
    auto ck = [&](cudaError_t e, const char* what) {
        if (e != cudaSuccess) { *why = std::string(what) + ": " + cudaGetErrorString(e); return false; }
        return true;
    };
    // flags: [0] written by the up neighbour, [1] by the down neighbour, [2] wait-timeout flag (own)
    if (!ck(cudaMalloc((void**)&c->flags, 24), "flags") || !ck(cudaMemset(c->flags, 0, 24), "flags")) return false;
    Blob mine{};
    for (int p = 0; p < c->nplanes; ++p)
        if (!ck(cudaIpcGetMemHandle(&mine.planes[p], c->planes[p]), "cudaIpcGetMemHandle(plane)")) return false;
    if (!ck(cudaIpcGetMemHandle(&mine.flags, c->flags), "cudaIpcGetMemHandle(flags)")) return false;
    mine.rows = c->g.My_local;
    // planes must never be reallocated or swapped from now on (set_config copies, see swap_in_spare)
    for (int p = 0; p < c->nplanes; ++p)
        if (!c->spare[p] && !ck(cudaMalloc((void**)&c->spare[p], (size_t)c->plane_words * 8), "spare planes")) return false;
    uint8_t* dsend = nullptr;
    uint8_t* drecv = nullptr;
    if (!ck(cudaMalloc((void**)&dsend, sizeof(Blob)), "blob") ||
        !ck(cudaMalloc((void**)&drecv, sizeof(Blob) * (size_t)c->world), "blobs")) { cudaFree(dsend); return false; }
    std::vector<Blob> all((size_t)c->world);
    bool ok = ck(cudaMemcpy(dsend, &mine, sizeof(Blob), cudaMemcpyHostToDevice), "blob upload");
    if (ok) {
        const ncclResult_t r = g_nccl.AllGather(dsend, drecv, sizeof(Blob), ncclUint8, c->comm, c->stream);
        if (r != ncclSuccess) { *why = std::string("ncclAllGather: ") + g_nccl.GetErrorString(r); ok = false; }
    }
    ok = ok && ck(cudaStreamSynchronize(c->stream), "all-gather");
    ok = ok && ck(cudaMemcpy(all.data(), drecv, sizeof(Blob) * (size_t)c->world, cudaMemcpyDeviceToHost), "blob download");
    cudaFree(dsend);
    cudaFree(drecv);
    if (!ok) return false;
    if (c->rank_up == c->rank) {
        // NCCL loopback (a one-rank ring): the neighbour is this rank -- its own planes and flags
        // (CUDA IPC cannot map a handle in the process that exported it); same kernels, same flags
        for (int p = 0; p < c->nplanes; ++p) c->peer_up[p] = c->peer_dn[p] = c->planes[p];
        c->peer_up_flags = c->peer_dn_flags = c->flags;
        c->peer_up_rows = (int)all[(size_t)c->rank].rows;
        c->fused = c->fused_ipc = true;
        return true;
    }
    auto open = [&](const cudaIpcMemHandle_t& hnd, void** ptr) {
        return ck(cudaIpcOpenMemHandle(ptr, hnd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle") &&
               (c->ipc_open.push_back(*ptr), true);
    };
    const Blob& up = all[(size_t)c->rank_up];
    const Blob& dn = all[(size_t)c->rank_down];
    void* ptr = nullptr;
    for (int p = 0; p < c->nplanes; ++p) {
        if (!open(up.planes[p], &ptr)) return false;
        c->peer_up[p] = (uint64_t*)ptr;
        if (c->rank_down == c->rank_up) c->peer_dn[p] = c->peer_up[p];   // world 2: one mapping
        else { if (!open(dn.planes[p], &ptr)) return false; c->peer_dn[p] = (uint64_t*)ptr; }
    }
    if (!open(up.flags, &ptr)) return false;
    c->peer_up_flags = (unsigned long long*)ptr;
    if (c->rank_down == c->rank_up) c->peer_dn_flags = c->peer_up_flags;
    else { if (!open(dn.flags, &ptr)) return false; c->peer_dn_flags = (unsigned long long*)ptr; }
    c->peer_up_rows = (int)up.rows;
    c->fused = c->fused_ipc = true;
    return true;
}

static kmc_status create_ctx(const kmc_geometry* geom, const kmc_model* model, const kmc_dist* dist, bool vgroup,
                             kmc_ctx** out) {
    if (!out) return fail(nullptr, KMC_EINVAL, "NULL out");
    *out = nullptr;
    if (!geom || !model) return fail(nullptr, KMC_EINVAL, "NULL geometry or model");
    if (model->kind < 0 || model->kind > 4) return fail(nullptr, KMC_EINVAL, "unknown model kind %d", model->kind);
    if (geom->ndim != 1 && geom->ndim != 2) return fail(nullptr, KMC_EINVAL, "ndim must be 1 or 2");
    if (geom->replicas < 1) return fail(nullptr, KMC_EINVAL, "replicas must be >= 1");
    const int world = dist ? dist->world : 1, rank = dist ? dist->rank : 0;
    if (world < 1 || rank < 0 || rank >= world) return fail(nullptr, KMC_EINVAL, "bad rank/world");
    // NCCL loopback (kmc.h, kmc_dist): world = 1 with an NCCL unique id runs a 2D lattice as a
    // one-rank periodic ring through the multi-GPU data plane -- ghost rows, NCCL send/recv to self
    // (or the fused exchange with device flags) -- so that transport executes on a single GPU
    const bool loopback = !vgroup && world == 1 && dist && dist->nccl_unique_id && geom->ndim == 2;

    const int ndim = geom->ndim;
    const long long H = ndim == 1 ? 1 : geom->dims[0];
    const long long W = ndim == 1 ? geom->dims[0] : geom->dims[1];
    const int qy = ndim == 1 ? 1 : geom->cell[0];
    const int qx = ndim == 1 ? geom->cell[0] : geom->cell[1];
    const bool cross = model->kind != KMC_ADSDES;
    if (H < 1 || W < 1 || qx < 1 || qy < 1) return fail(nullptr, KMC_EINVAL, "dims and cell must be positive");
    if (qx * qy > 64) return fail(nullptr, KMC_EPARTITION, "cell has %d sites (> 64)", qx * qy);
    if (W % qx || H % qy) return fail(nullptr, KMC_EPARTITION, "dims not divisible by the cell");
    const long long Mx = W / qx, My = H / qy;
    if (Mx % 2 || (ndim == 2 && My % 2)) return fail(nullptr, KMC_EPARTITION, "need an even number of cells per axis");
    if (cross && (qx < 2 || (ndim == 2 && qy < 2)))
        return fail(nullptr, KMC_EPARTITION, "cross-cell-writing model needs cell extent >= 2 (R7)");
    int C = geom->colours;
    if (C == 0) C = (ndim == 1 || !cross) ? 2 : 4;
    if (C != 2 && C != 4) return fail(nullptr, KMC_EPARTITION, "colours must be 2 or 4");
    if (ndim == 1 && C != 2) return fail(nullptr, KMC_EPARTITION, "1D lattices use 2 colours");
    if (ndim == 2 && cross && C == 2)
        return fail(nullptr, KMC_EPARTITION, "2D model with cross-cell writes needs 4 colours (R6)");
    if ((long long)geom->replicas * Mx * My > 0xFFFFFFFFLL)
        return fail(nullptr, KMC_EPARTITION, "more than 2^32 cells in total (Philox counter word)");
    int64_t plan[6];
    if (dist && dist->row_bounds && ndim == 2 && world > 1) {
        // caller-chosen slabs (f4 re-partition): world+1 cell-row bounds, each slab an even number
        // (>= 2) of cell rows so the colour pattern stays global
        const int64_t* b = dist->row_bounds;
        if (b[0] != 0 || b[world] != My)
            return fail(nullptr, KMC_EPARTITION, "row_bounds must run from 0 to %lld cell rows", (long long)My);
        for (int r = 0; r < world; ++r)
            if (b[r + 1] - b[r] < 2 || (b[r + 1] - b[r]) % 2)
                return fail(nullptr, KMC_EPARTITION, "row_bounds: slab %d has %lld cell rows (need an even number >= 2)",
                            r, (long long)(b[r + 1] - b[r]));
        plan[0] = 0; plan[1] = geom->replicas; plan[2] = b[rank]; plan[3] = b[rank + 1] - b[rank];
        plan[4] = (rank + world - 1) % world; plan[5] = (rank + 1) % world;
    } else {
        kmc_status ps = kmc_partition_plan(geom, model->kind, world, rank, plan);
        if (ps != KMC_OK) return ps;
    }
    if (loopback) plan[4] = plan[5] = 0;                     // a ring of one: both neighbours are rank 0

    kmc_ctx* c = new kmc_ctx();
    c->geom = *geom;
    c->model = *model;
    c->rank = rank; c->world = world; c->device = dist ? dist->device : 0;
    c->kind = model->kind;
    c->nplanes = (model->kind >= KMC_ZGB) ? 2 : 1;
    c->nstates = c->nplanes + 1;
    c->C = C;
    c->cross = cross;
    c->W = W;
    Geo& g = c->g;
    g.ndim = ndim; g.qx = qx; g.qy = qy; g.nsite = qx * qy;
    g.Mx = (int)Mx;
    g.R = (int)plan[1];
    g.rep_offset = (int)plan[0];
    g.row_offset = (int)plan[2];
    g.My_local = (int)plan[3];
    g.ghost = ((world > 1 || loopback) && ndim == 2) ? 1 : 0;
    g.M_global = Mx * My;
    g.shN = qx * (qy - 1);
    g.valid = lowmask(qx * qy);
    g.col0 = 0; g.colL = 0;
    for (int y = 0; y < qy; ++y) { g.col0 |= 1ull << (y * qx); g.colL |= 1ull << (y * qx + qx - 1); }
    g.row0 = lowmask(qx);
    g.rowL = g.row0 << g.shN;
    g.notcol0 = g.valid & ~g.col0;
    g.notcolL = g.valid & ~g.colL;
    g.notrow0 = g.valid & ~g.row0;
    g.notrowL = g.valid & ~g.rowL;
    c->H_local = (long long)g.My_local * qy;
    c->rank_up = (int)plan[4];
    c->rank_down = (int)plan[5];
    if (ndim == 2) {   // every rank's slab bounds (the same on every rank: collective checks, f3)
        c->bounds.resize((size_t)world + 1);
        for (int r = 0; r <= world; ++r)
            c->bounds[(size_t)r] = (dist && dist->row_bounds && world > 1) ? dist->row_bounds[r] : (int64_t)r * (My / world);
    }

    // a1: the rate table
    c->nclass = build_classes(*model, ndim, c->ctype, c->cdir, c->ckappa, c->crate);
    c->F = quantise(c->crate, c->nclass, (long long)g.nsite * types_per_site(c->kind, 2 * ndim), c->crate_u64);
    if (c->F < 0) { delete c; return fail(nullptr, KMC_EINVAL, "rates must be finite and >= 0 (and quantisable)"); }
    {   // kernel-choice heuristic: sites x mean class rate ~ events per unit time per cell
        double s = 0.0;
        for (int i = 0; i < c->nclass; ++i) s += c->crate[i];
        c->rate_per_cell = (double)g.nsite * s / (double)c->nclass;
    }

    cudaError_t e = cudaSetDevice(c->device);
    if (e != cudaSuccess) { delete c; return fail(nullptr, KMC_ECUDA, "cudaSetDevice(%d): %s", dist ? dist->device : 0, cudaGetErrorString(e)); }
    if (dist && dist->stream) c->stream = (cudaStream_t)dist->stream;
    else {
        e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) { delete c; return fail(nullptr, KMC_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e)); }
        c->own_stream = true;
    }
    const long long rows_storage = g.My_local + 2 * g.ghost;
    c->plane_words = rows_storage * (long long)g.R * g.Mx;
    const long long owned = (long long)g.My_local * g.R * g.Mx;
    auto alloc = [&](void** p, size_t n) -> bool { return cudaMalloc(p, n) == cudaSuccess; };
    bool ok = true;
    for (int p = 0; p < c->nplanes; ++p) ok = ok && alloc((void**)&c->planes[p], (size_t)c->plane_words * 8);
    ok = ok && alloc((void**)&c->wev, (size_t)owned * 4);
    ok = ok && alloc((void**)&c->wmark, (size_t)owned * 4);
    ok = ok && alloc((void**)&c->ev_total, 8);
    ok = ok && alloc((void**)&c->queue, 8) && cudaMemsetAsync(c->queue, 0, 8, c->stream) == cudaSuccess;
    ok = ok && alloc((void**)&c->obs_buf, KMC_OBS_WORDS * 8);
    ok = ok && alloc((void**)&c->logtab, kLogTab * sizeof(double2));
    if (ok) {   // log_spec tables, host libm; uploaded once
        double2 bucket[kLogBuckets], tab[kLogTab];
        for (int j = 0; j < kLogBuckets; ++j) {
            bucket[j].x = 128.0 / (double)(j + 91);
            bucket[j].y = -std::log(bucket[j].x);
        }
        // entry i -> bucket j = round(128 m) - 91 of the mantissas with high bits t:
        // not halved (t <= 0x6A, i = t): j = 128 + ((t + 1) >> 1) - 91; halved (i = t + 1, t >= 0x6A):
        // j = 64 + ((t + 2) >> 2) - 91.  Both stay in [0, 90].
        // Halved entries hold c_j / 2 (exact): log_spec multiplies the unhalved mantissa by them,
        // (2m) (c_j / 2) = m c_j exactly, so r = fma(., ., -1) rounds the same real number.
        for (int i = 0; i < kLogTab; ++i) {
            tab[i] = bucket[i <= 0x6A ? 37 + ((i + 1) >> 1) : ((i + 1) >> 2) - 27];
            if (i > 0x6A) tab[i].x *= 0.5;
        }
        ok = cudaMemcpy(c->logtab, tab, sizeof tab, cudaMemcpyHostToDevice) == cudaSuccess;
    }
    ok = ok && alloc((void**)&c->obs_acc, (kObsCounters + 1) * 8) &&
         cudaMemsetAsync(c->obs_acc, 0, (kObsCounters + 1) * 8, c->stream) == cudaSuccess;
    ok = ok && alloc((void**)&c->err_flag, 4);
    if (g.ghost) {
        ok = ok && alloc((void**)&c->ghost_snap, (size_t)4 * g.R * g.Mx * 8);
        ok = ok && alloc((void**)&c->ghost_recv, (size_t)4 * g.R * g.Mx * 8);
    }
    ok = ok && cudaHostAlloc((void**)&c->h_obs, KMC_OBS_WORDS * 8, cudaHostAllocMapped) == cudaSuccess &&
         cudaHostGetDevicePointer((void**)&c->d_hobs, c->h_obs, 0) == cudaSuccess;
    ok = ok && cudaMallocHost((void**)&c->h_flag, 8) == cudaSuccess;
    ok = ok && cudaMallocHost((void**)&c->h_err, 4) == cudaSuccess;
    if (!ok) { kmc_destroy(c); return fail(nullptr, KMC_ENOMEM, "device allocation failed (%lld words)", c->plane_words); }
    for (int p = 0; p < c->nplanes; ++p) cudaMemsetAsync(c->planes[p], 0, (size_t)c->plane_words * 8, c->stream);
    cudaMemsetAsync(c->wev, 0, (size_t)owned * 4, c->stream);
    cudaMemsetAsync(c->wmark, 0, (size_t)owned * 4, c->stream);
    cudaMemsetAsync(c->ev_total, 0, 8, c->stream);
    e = cudaStreamSynchronize(c->stream);
    if (e != cudaSuccess) { kmc_destroy(c); return fail(nullptr, KMC_ECUDA, "init: %s", cudaGetErrorString(e)); }

    c->vgroup = vgroup;
    build_args_template(c);
    if ((world > 1 || loopback) && !vgroup) {
        std::string why;
        if (!dist->nccl_unique_id) { kmc_destroy(c); return fail(nullptr, KMC_EINVAL, "world > 1 needs nccl_unique_id"); }
        if (!load_nccl(&why)) { kmc_destroy(c); return fail(nullptr, KMC_ENCCL, "%s", why.c_str()); }
        ncclUniqueId id;
        memcpy(&id, dist->nccl_unique_id, 128);
        ncclResult_t r = g_nccl.CommInitRank(&c->comm, world, id, rank);
        if (r != ncclSuccess) { kmc_destroy(c); return fail(nullptr, KMC_ENCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r)); }
        if (dist->fused_exchange && ndim == 2) {   // (world 1: the loopback ring)
            std::string why2;
            if (!setup_fused_ipc(c, &why2)) { kmc_destroy(c); return fail(nullptr, KMC_ECUDA, "fused exchange setup: %s", why2.c_str()); }
        }
    }
    *out = c;
    return KMC_OK;
}

extern "C" {

void kmc_destroy(kmc_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    // fused exchange across GPUs: the neighbours' last windows write into our rows; wait for their
    // completion signals before the buffers go away
    if (c->fused_ipc && c->flags && c->stream) launch_wait_flags(c->flags, c->epoch, c->stream);
    if (c->stream) cudaStreamSynchronize(c->stream);
    if (c->copy_stream) { cudaStreamSynchronize(c->copy_stream); cudaStreamDestroy(c->copy_stream); }
    if (c->dl_stream) { cudaStreamSynchronize(c->dl_stream); cudaStreamDestroy(c->dl_stream); }
    if (c->staged_ev) cudaEventDestroy(c->staged_ev);
    if (c->consumed_ev) cudaEventDestroy(c->consumed_ev);
    if (c->dl_ev) cudaEventDestroy(c->dl_ev);
    if (c->dl_start_ev) cudaEventDestroy(c->dl_start_ev);
    if (c->h_stage_err) cudaFreeHost(c->h_stage_err);
    for (void* p : c->ipc_open) cudaIpcCloseMemHandle(p);
    if (c->comm && g_nccl.CommDestroy) g_nccl.CommDestroy(c->comm);
    if (!c->borrowed)
        for (int p = 0; p < 2; ++p) cudaFree(c->planes[p]);
    cudaFree(c->flags);
    cudaFree(c->wev); cudaFree(c->wmark); cudaFree(c->strips); cudaFree(c->wl_out); cudaFree(c->ev_total); cudaFree(c->queue); cudaFree(c->obs_buf); cudaFree(c->obs_acc); cudaFree(c->logtab); cudaFree(c->err_flag);
    cudaFree(c->staging); cudaFree(c->ghost_snap); cudaFree(c->ghost_recv); cudaFree(c->series);
    cudaFree(c->spare[0]); cudaFree(c->spare[1]); cudaFree(c->spare2[0]); cudaFree(c->spare2[1]);
    if (c->h_obs) cudaFreeHost(c->h_obs);
    if (c->h_flag) cudaFreeHost(c->h_flag);
    if (c->h_err) cudaFreeHost(c->h_err);
    for (auto& pr : c->tev) { cudaEventDestroy(pr.first); cudaEventDestroy(pr.second); }
    if (c->own_stream) cudaStreamDestroy(c->stream);
    if (c->vg_shared && --c->vg_shared->refs == 0) {
        cudaStreamDestroy(c->vg_shared->stream);
        delete c->vg_shared;
    }
    cudaGetLastError();   // teardown is best effort: do not leave a stale error for the next call
    delete c;
}

kmc_status kmc_local_shape(const kmc_ctx* c, int64_t* rl, int64_t* hl, int64_t* w, int64_t* ro, int64_t* yo) {
    if (!c) return KMC_EINVAL;
    if (rl) *rl = c->g.R;
    if (hl) *hl = c->H_local;
    if (w) *w = c->W;
    if (ro) *ro = c->g.rep_offset;
    if (yo) *yo = (int64_t)c->g.row_offset * c->g.qy;
    return KMC_OK;
}

// A validated configuration in the spare planes becomes the lattice.  Normally a pointer swap; with
// the fused exchange the plane buffers are mapped by the neighbour ranks, so they must stay put.
static kmc_status swap_in_spare(kmc_ctx* c) {
    kmc_status sq = fused_quiesce(c);
    const bool in_place = c->fused || c->borrowed;   // mapped by the neighbours / the caller's buffer
    if (sq == KMC_OK && in_place) sq = dl_guard(c, c->planes[0]);   // copied into the planes in place
    if (sq != KMC_OK) return sq;
    for (int p = 0; p < c->nplanes; ++p) {
        if (in_place)
            CUDA_TRY(c, launch_copy_u64(c->planes[p], c->spare[p], c->plane_words, c->stream));
        else
            std::swap(c->spare[p], c->planes[p]);
    }
    return KMC_OK;
}

kmc_status kmc_planes_layout(const kmc_ctx* c, int32_t* planes, int64_t* words_per_plane, int64_t* storage_rows,
                             int32_t* ghost) {
    if (!c) return KMC_EINVAL;
    if (planes) *planes = c->nplanes;
    if (words_per_plane) *words_per_plane = c->plane_words;
    if (storage_rows) *storage_rows = c->g.My_local + 2 * c->g.ghost;
    if (ghost) *ghost = c->g.ghost;
    return KMC_OK;
}

kmc_status kmc_attach_planes(kmc_ctx* c, uint64_t* dev, int64_t nwords) {
    if (!c || !dev) return fail(c, KMC_EINVAL, "NULL argument");
    if (((uintptr_t)dev & 7u) != 0) return fail(c, KMC_EINVAL, "dev_planes must be 8-byte aligned");
    if (nwords != (int64_t)c->nplanes * c->plane_words)
        return fail(c, KMC_EINVAL, "nwords %lld != %d planes x %lld words", (long long)nwords, c->nplanes, c->plane_words);
    if (c->fused) return fail(c, KMC_ESTATE, "borrowed planes with the fused exchange (IPC mappings made at create)");
    if (c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st = dl_guard(c, c->planes[0]);
    if (st != KMC_OK) return st;
    if (c->dl_pending) CUDA_TRY(c, cudaEventSynchronize(c->dl_ev));   // a download reads the old planes
    c->dl_pending = false;
    uint64_t* old[2] = {c->planes[0], c->planes[1]};
    for (int p = 0; p < c->nplanes; ++p)
        CUDA_TRY(c, cudaMemcpyAsync(dev + (size_t)p * c->plane_words, old[p], (size_t)c->plane_words * 8,
                                    cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int p = 0; p < c->nplanes; ++p) {
        if (!c->borrowed) cudaFree(old[p]);
        c->planes[p] = dev + (size_t)p * c->plane_words;
    }
    c->borrowed = true;
    return KMC_OK;
}

static long long slab_bytes(const kmc_ctx* c) { return (long long)c->g.R * c->H_local * c->W; }

static kmc_status ensure_staging(kmc_ctx* c) {
    if (c->staging) return KMC_OK;
    if (cudaMalloc((void**)&c->staging, (size_t)slab_bytes(c)) != cudaSuccess)
        return fail(c, KMC_ENOMEM, "staging allocation of %lld bytes failed", slab_bytes(c));
    return KMC_OK;
}

kmc_status kmc_set_config_device(kmc_ctx* c, const uint8_t* dev, int64_t nbytes) {
    if (c && c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    if (!c || !dev) return fail(c, KMC_EINVAL, "NULL argument");
    if (nbytes != slab_bytes(c)) return fail(c, KMC_EINVAL, "nbytes %lld != local slab %lld", (long long)nbytes, slab_bytes(c));
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sq = fused_quiesce(c);
    if (sq == KMC_OK) sq = dl_guard(c, c->planes[0]);
    if (sq != KMC_OK) return sq;
    CUDA_TRY(c, cudaMemsetAsync(c->err_flag, 0, 4, c->stream));   // kmc_device_errors reports this upload
    CUDA_TRY(c, launch_pack(c->g, dev, c->planes[0], c->nplanes > 1 ? c->planes[1] : nullptr, c->nstates, c->err_flag, c->stream));
    return KMC_OK;
}

kmc_status kmc_get_config_device(kmc_ctx* c, uint8_t* dev, int64_t nbytes) {
    if (!c || !dev) return fail(c, KMC_EINVAL, "NULL argument");
    if (nbytes != slab_bytes(c)) return fail(c, KMC_EINVAL, "nbytes %lld != local slab %lld", (long long)nbytes, slab_bytes(c));
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sq = fused_quiesce(c);
    if (sq != KMC_OK) return sq;
    CUDA_TRY(c, launch_unpack(c->g, c->planes[0], c->planes[1], c->nplanes, dev, c->stream));
    return KMC_OK;
}

kmc_status kmc_init_random(kmc_ctx* c, const double* probs, int32_t nprobs, uint64_t seed) {
    if (!c || !probs) return fail(c, KMC_EINVAL, "NULL argument");
    if (c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    if (nprobs != c->nstates) return fail(c, KMC_EINVAL, "need %d probabilities, got %d", c->nstates, nprobs);
    unsigned long long thr[2] = {0, 0};
    double cum = 0.0;
    for (int j = 0; j < nprobs; ++j)
        if (!(probs[j] >= 0.0) || std::isinf(probs[j])) return fail(c, KMC_EINVAL, "probabilities must be finite and >= 0");
    for (int j = 0; j + 1 < nprobs; ++j) {   // R32: T_j = floor(2^32 (p_0 + .. + p_j)), 2^32 once the sum reaches 1
        cum = cum + probs[j];
        if (cum > 1.0 + 1e-12) return fail(c, KMC_EINVAL, "partial sums of the probabilities exceed 1");
        thr[j] = cum >= 1.0 ? (1ull << 32) : (unsigned long long)std::floor(cum * 4294967296.0);
    }
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sq = fused_quiesce(c);
    if (sq == KMC_OK) sq = dl_guard(c, c->planes[0]);
    if (sq != KMC_OK) return sq;
    CUDA_TRY(c, launch_init_random(c->g, c->planes[0], c->nplanes > 1 ? c->planes[1] : nullptr, seed, thr,
                                   nprobs - 1, c->stream));
    return KMC_OK;
}

kmc_status kmc_set_config(kmc_ctx* c, const uint8_t* host, int64_t nbytes) {
    if (c && c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nbytes != slab_bytes(c)) return fail(c, KMC_EINVAL, "nbytes %lld != local slab %lld", (long long)nbytes, slab_bytes(c));
    kmc_status st = ensure_staging(c);
    if (st != KMC_OK) return st;
    CUDA_TRY(c, cudaSetDevice(c->device));
    // validate in a scratch copy of the planes so an invalid slab leaves the lattice unchanged
    CUDA_TRY(c, cudaMemsetAsync(c->err_flag, 0, 4, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->staging, host, (size_t)nbytes, cudaMemcpyHostToDevice, c->stream));
    // persistent spare planes (allocated once): pack there, swap in only if every spin was valid
    for (int p = 0; p < c->nplanes; ++p)
        if (!c->spare[p] && cudaMalloc((void**)&c->spare[p], (size_t)c->plane_words * 8) != cudaSuccess)
            return fail(c, KMC_ENOMEM, "spare plane allocation failed");
    st = fused_quiesce(c);
    if (st == KMC_OK) st = dl_guard(c, c->spare[0]);
    if (st != KMC_OK) return st;
    if (c->g.ghost)   // ghost rows are refreshed by the next exchange; keep them defined
        for (int p = 0; p < c->nplanes; ++p)
            CUDA_TRY(c, cudaMemcpyAsync(c->spare[p], c->planes[p], (size_t)c->plane_words * 8, cudaMemcpyDeviceToDevice, c->stream));
    CUDA_TRY(c, launch_pack(c->g, c->staging, c->spare[0], c->spare[1], c->nstates, c->err_flag, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->err_flag, 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (*c->h_err) return fail(c, KMC_EINVAL, "spin value >= %d in the configuration", c->nstates);
    return swap_in_spare(c);
}

kmc_status kmc_get_config(kmc_ctx* c, uint8_t* host, int64_t nbytes) {
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nbytes != slab_bytes(c)) return fail(c, KMC_EINVAL, "nbytes %lld != local slab %lld", (long long)nbytes, slab_bytes(c));
    kmc_status st = ensure_staging(c);
    if (st != KMC_OK) return st;
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sq = fused_quiesce(c);
    if (sq != KMC_OK) return sq;
    CUDA_TRY(c, launch_unpack(c->g, c->planes[0], c->planes[1], c->nplanes, c->staging, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(host, c->staging, (size_t)nbytes, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return KMC_OK;
}

// Bit-packed slab: [plane][owned cell row][replica][cx] u64 words, exactly the owned rows of the
// device planes, so H2D / D2H are one contiguous copy per plane (8x fewer bytes than uint8 sites).
static long long packed_words(const kmc_ctx* c) { return (long long)c->nplanes * c->g.My_local * c->g.R * c->g.Mx; }
static kmc_status ensure_copy_stream(kmc_ctx* c);

kmc_status kmc_set_config_packed(kmc_ctx* c, const uint64_t* host, int64_t nwords) {
    if (c && c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nwords != packed_words(c)) return fail(c, KMC_EINVAL, "nwords %lld != packed local slab %lld", (long long)nwords, packed_words(c));
    CUDA_TRY(c, cudaSetDevice(c->device));
    for (int p = 0; p < c->nplanes; ++p)
        if (!c->spare[p] && cudaMalloc((void**)&c->spare[p], (size_t)c->plane_words * 8) != cudaSuccess)
            return fail(c, KMC_ENOMEM, "spare plane allocation failed");
    const size_t owned = (size_t)c->g.My_local * c->g.R * c->g.Mx;
    const size_t off = (size_t)c->g.ghost * c->g.R * c->g.Mx;
    CUDA_TRY(c, cudaMemsetAsync(c->err_flag, 0, 4, c->stream));
    kmc_status sq = fused_quiesce(c);
    if (sq == KMC_OK) sq = dl_guard(c, c->spare[0]);
    if (sq != KMC_OK) return sq;
    for (int p = 0; p < c->nplanes; ++p) {
        if (c->g.ghost)   // ghost rows are refreshed by the next exchange; keep them defined
            CUDA_TRY(c, cudaMemcpyAsync(c->spare[p], c->planes[p], (size_t)c->plane_words * 8, cudaMemcpyDeviceToDevice, c->stream));
        CUDA_TRY(c, cudaMemcpyAsync(c->spare[p] + off, host + (size_t)p * owned, owned * 8, cudaMemcpyHostToDevice, c->stream));
    }
    CUDA_TRY(c, launch_check_packed(c->spare[0] + off, c->nplanes > 1 ? c->spare[1] + off : nullptr, (long long)owned,
                                    c->g.valid, c->err_flag, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(c->h_err, c->err_flag, 4, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (*c->h_err) return fail(c, KMC_EINVAL, "packed configuration has bits outside the cells or a site both CO and O");
    return swap_in_spare(c);
}

kmc_status kmc_stage_config_packed(kmc_ctx* c, const uint64_t* host, int64_t nwords) {
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nwords != packed_words(c)) return fail(c, KMC_EINVAL, "nwords %lld != packed local slab %lld", (long long)nwords, packed_words(c));
    if (c->staged) return fail(c, KMC_ESTATE, "a staged configuration is pending (kmc_commit_config first)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sc = ensure_copy_stream(c);
    if (sc != KMC_OK) return sc;
    for (int p = 0; p < c->nplanes; ++p)
        if (!c->spare[p] && cudaMalloc((void**)&c->spare[p], (size_t)c->plane_words * 8) != cudaSuccess)
            return fail(c, KMC_ENOMEM, "spare plane allocation failed");
    const size_t owned = (size_t)c->g.My_local * c->g.R * c->g.Mx;
    const size_t off = (size_t)c->g.ghost * c->g.R * c->g.Mx;
    cudaStream_t cs = c->copy_stream;
    // a pending download (its own stream) may still read the spare planes -- the planes current
    // before the last commit: stage into a third buffer instead, so that the upload overlaps the
    // download (buffers rotate current -> downloading -> staging)
    if (c->dl_pending && c->dl_buf == c->spare[0]) {
        for (int p = 0; p < c->nplanes; ++p)
            if (!c->spare2[p] && cudaMalloc((void**)&c->spare2[p], (size_t)c->plane_words * 8) != cudaSuccess)
                return fail(c, KMC_ENOMEM, "third plane buffer allocation failed");
        for (int p = 0; p < c->nplanes; ++p) std::swap(c->spare[p], c->spare2[p]);
    }
    // the spare planes were current before an earlier commit: the windows enqueued before the last
    // commit may still read them
    if (c->consumed_valid) CUDA_TRY(c, cudaStreamWaitEvent(cs, c->consumed_ev, 0));
    *(volatile unsigned int*)c->h_stage_err = 0u;     // the previous staged check has completed (commit)
    for (int p = 0; p < c->nplanes; ++p)
        CUDA_TRY(c, cudaMemcpyAsync(c->spare[p] + off, host + (size_t)p * owned, owned * 8, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(c, launch_check_packed(c->spare[0] + off, c->nplanes > 1 ? c->spare[1] + off : nullptr, (long long)owned,
                                    c->g.valid, c->stage_err, cs));
    CUDA_TRY(c, cudaEventRecord(c->staged_ev, cs));
    c->staged = true;
    return KMC_OK;
}

kmc_status kmc_commit_config(kmc_ctx* c) {
    if (!c) return KMC_EINVAL;
    if (!c->staged) return fail(c, KMC_ESTATE, "no staged configuration (kmc_stage_config_packed first)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaEventSynchronize(c->staged_ev));         // normally long done: it overlapped the windows
    c->staged = false;
    if (*(volatile unsigned int*)c->h_stage_err)
        return fail(c, KMC_EINVAL, "staged packed configuration has bits outside the cells or a site both CO and O (discarded)");
    CUDA_TRY(c, cudaStreamWaitEvent(c->stream, c->staged_ev, 0));
    kmc_status sq = fused_quiesce(c);
    if (sq == KMC_OK && c->g.ghost) sq = dl_guard(c, c->spare[0]);   // the ghost-row copies below write the spare
    if (sq != KMC_OK) return sq;
    if (c->g.ghost) {   // ghost rows are refreshed by the next exchange; keep them defined (stream-ordered)
        const size_t row = (size_t)c->g.R * c->g.Mx, last = (size_t)(c->g.My_local + 1) * row;
        for (int p = 0; p < c->nplanes; ++p) {
            CUDA_TRY(c, launch_copy_u64(c->spare[p], c->planes[p], (long long)row, c->stream));
            CUDA_TRY(c, launch_copy_u64(c->spare[p] + last, c->planes[p] + last, (long long)row, c->stream));
        }
    }
    kmc_status st = swap_in_spare(c);
    if (st != KMC_OK) return st;
    CUDA_TRY(c, cudaEventRecord(c->consumed_ev, c->stream));
    c->consumed_valid = true;
    return KMC_OK;
}

static kmc_status ensure_copy_stream(kmc_ctx* c) {
    if (c->copy_stream) return KMC_OK;
    CUDA_TRY(c, cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->staged_ev, cudaEventDisableTiming));
    CUDA_TRY(c, cudaEventCreateWithFlags(&c->consumed_ev, cudaEventDisableTiming));
    if (cudaHostAlloc((void**)&c->h_stage_err, 4, cudaHostAllocMapped) != cudaSuccess ||
        cudaHostGetDevicePointer((void**)&c->stage_err, c->h_stage_err, 0) != cudaSuccess)
        return fail(c, KMC_ENOMEM, "staging flag allocation failed");
    return KMC_OK;
}

kmc_status kmc_download_config_packed(kmc_ctx* c, uint64_t* host, int64_t nwords) {
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nwords != packed_words(c)) return fail(c, KMC_EINVAL, "nwords %lld != packed local slab %lld", (long long)nwords, packed_words(c));
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st = ensure_copy_stream(c);
    if (st != KMC_OK) return st;
    if (!c->dl_ev) {
        CUDA_TRY(c, cudaStreamCreateWithFlags(&c->dl_stream, cudaStreamNonBlocking));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->dl_ev, cudaEventDisableTiming));
        CUDA_TRY(c, cudaEventCreateWithFlags(&c->dl_start_ev, cudaEventDisableTiming));
    }
    if (c->dl_pending) CUDA_TRY(c, cudaEventSynchronize(c->dl_ev));   // one download at a time
    st = fused_quiesce(c);
    if (st != KMC_OK) return st;
    // the copy starts after everything enqueued on the context's stream so far
    CUDA_TRY(c, cudaEventRecord(c->dl_start_ev, c->stream));
    CUDA_TRY(c, cudaStreamWaitEvent(c->dl_stream, c->dl_start_ev, 0));
    const size_t owned = (size_t)c->g.My_local * c->g.R * c->g.Mx;
    const size_t off = (size_t)c->g.ghost * c->g.R * c->g.Mx;
    for (int p = 0; p < c->nplanes; ++p)
        CUDA_TRY(c, cudaMemcpyAsync(host + (size_t)p * owned, c->planes[p] + off, owned * 8, cudaMemcpyDeviceToHost,
                                    c->dl_stream));
    CUDA_TRY(c, cudaEventRecord(c->dl_ev, c->dl_stream));
    c->dl_pending = true;
    c->dl_buf = c->planes[0];
    return KMC_OK;
}

kmc_status kmc_download_wait(kmc_ctx* c) {
    if (!c) return KMC_EINVAL;
    if (!c->dl_ev) return KMC_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaEventSynchronize(c->dl_ev));
    c->dl_pending = false;
    return KMC_OK;
}

kmc_status kmc_get_config_packed(kmc_ctx* c, uint64_t* host, int64_t nwords) {
    if (!c || !host) return fail(c, KMC_EINVAL, "NULL argument");
    if (nwords != packed_words(c)) return fail(c, KMC_EINVAL, "nwords %lld != packed local slab %lld", (long long)nwords, packed_words(c));
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status sq = fused_quiesce(c);
    if (sq != KMC_OK) return sq;
    const size_t owned = (size_t)c->g.My_local * c->g.R * c->g.Mx;
    const size_t off = (size_t)c->g.ghost * c->g.R * c->g.Mx;
    for (int p = 0; p < c->nplanes; ++p)
        CUDA_TRY(c, cudaMemcpyAsync(host + (size_t)p * owned, c->planes[p] + off, owned * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return KMC_OK;
}

kmc_status kmc_substep(kmc_ctx* c, int32_t colour, double duration) {
    if (!c) return KMC_EINVAL;
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: use kmc_vgroup_run");
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st = fused_refresh(c);
    if (st != KMC_OK) return st;
    return do_substep(c, colour, duration);
}

kmc_status kmc_run(kmc_ctx* c, double T, double dt, kmc_scheme scheme) {
    if (!c) return KMC_EINVAL;
    if (!(dt > 0.0) || !(T >= 0.0) || std::isinf(T)) return fail(c, KMC_EINVAL, "need dt > 0 and finite T >= 0");
    if (scheme < KMC_LIE || scheme > KMC_RANDOM) return fail(c, KMC_EINVAL, "unknown scheme %d", (int)scheme);
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: use kmc_vgroup_run");
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st0 = fused_refresh(c);
    if (st0 != KMC_OK) return st0;
    bool truncated = false;
    for (double d : macro_durations(T, dt, &truncated)) {
        for (const auto& sd : macro_schedule(scheme, c->C, d, c->geom.seed, c->window)) {
            kmc_status st = do_substep(c, sd.first, sd.second);
            if (st != KMC_OK) return st;
        }
        c->time += d;
        kmc_status sr = record_sample(c);
        if (sr != KMC_OK) return sr;
    }
    return truncated ? KMC_WTRUNCATED : KMC_OK;
}

kmc_status kmc_run_multiscale(kmc_ctx* c, double T, double dt, int32_t n_fast, kmc_scheme inner,
                              uint64_t fast_classes) {
    if (!c) return KMC_EINVAL;
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: multiscale runs are not grouped");
    if (!(dt > 0.0) || !(T >= 0.0) || std::isinf(T)) return fail(c, KMC_EINVAL, "need dt > 0 and finite T >= 0");
    if (n_fast < 1) return fail(c, KMC_EINVAL, "n_fast must be >= 1");
    if (inner < KMC_LIE || inner > KMC_RANDOM) return fail(c, KMC_EINVAL, "unknown inner scheme %d", (int)inner);
    const uint64_t all = c->nclass >= 64 ? ~0ull : ((1ull << c->nclass) - 1ull);
    if (fast_classes == 0)   // default: the hop mechanisms (R12 diffusion, ZGB CO diffusion)
        for (int i = 0; i < c->nclass; ++i)
            if (c->ctype[i] == T_HOP || c->ctype[i] == T_COHOP || c->ctype[i] == T_OHOP) fast_classes |= 1ull << i;
    fast_classes &= all;
    if (fast_classes == 0 || fast_classes == all)
        return fail(c, KMC_EINVAL, "multiscale needs a non-empty proper subset of fast classes");
    const uint64_t slow = all & ~fast_classes;
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st0 = fused_refresh(c);
    if (st0 != KMC_OK) return st0;
    bool truncated = false;
    for (double d : macro_durations(T, dt, &truncated)) {
        // eq.(strang3): e^{d/2 L_r} [e^{(d/N) L_f}]^N e^{d/2 L_r}, each factor split over colours
        const double h = d * 0.5, df = d / (double)n_fast;
        auto factor = [&](double dur, uint64_t mask) -> kmc_status {
            for (const auto& sd : macro_schedule(inner, c->C, dur, c->geom.seed, c->window)) {
                kmc_status st = do_substep(c, sd.first, sd.second, mask);
                if (st != KMC_OK) return st;
            }
            return KMC_OK;
        };
        kmc_status st = factor(h, slow);
        for (int i = 0; i < n_fast && st == KMC_OK; ++i) st = factor(df, fast_classes);
        if (st == KMC_OK) st = factor(h, slow);
        if (st != KMC_OK) return st;
        c->time += d;
        kmc_status sr = record_sample(c);
        if (sr != KMC_OK) return sr;
    }
    return truncated ? KMC_WTRUNCATED : KMC_OK;
}

kmc_status kmc_run_nested(kmc_ctx* c, double T, double dt, int32_t n_inner, kmc_scheme outer, kmc_scheme inner,
                          int32_t block) {
    if (!c) return KMC_EINVAL;
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: use kmc_vgroup_run_nested");
    kmc_status st = check_nested(c, T, dt, n_inner, outer, inner, block);
    if (st != KMC_OK) return st;
    CUDA_TRY(c, cudaSetDevice(c->device));
    st = fused_quiesce(c);             // the exchange below reads rows the neighbours' fused windows wrote
    if (st != KMC_OK) return st;
    bool truncated = false;
    for (double d : macro_durations(T, dt, &truncated)) {
        for (const auto& of : outer_factors(outer, d)) {
            // eq.(opdecomp2): e^{D L^o} ~ [inner cycle of duration D/n]^n.  One halo exchange per
            // outer factor: the ghost rows belong to the inactive outer colour throughout it.
            const Nest nest{of.first, block};
            st = exchange_forward(c);
            for (int k = 0; k < n_inner && st == KMC_OK; ++k)
                for (const auto& sd : macro_schedule(inner, c->C, of.second / (double)n_inner, c->geom.seed, c->window)) {
                    st = launch_window(c, sd.first, sd.second, ~0ull, &nest);
                    if (st != KMC_OK) break;
                }
            if (st == KMC_OK) st = exchange_reverse(c);
            if (st != KMC_OK) return st;
        }
        c->time += d;
        kmc_status sr = record_sample(c);
        if (sr != KMC_OK) return sr;
    }
    return truncated ? KMC_WTRUNCATED : KMC_OK;
}

// ---- f4: workload histogram and cdf re-partition (R29) ----
static long long strip_count(const kmc_ctx* c) {
    return c->g.ndim == 2 ? c->geom.dims[0] / c->g.qy : (long long)c->g.Mx;
}

static kmc_status ensure_strips(kmc_ctx* c, int parts) {
    const long long M = strip_count(c);
    if (c->strips_n < M) {
        cudaFree(c->strips);
        c->strips = nullptr;
        if (cudaMalloc((void**)&c->strips, (size_t)M * 16) != cudaSuccess) return fail(c, KMC_ENOMEM, "strip buffers");
        c->strips_n = M;
    }
    if (!c->wl_out && cudaMalloc((void**)&c->wl_out, (size_t)(4096 + 3) * 8) != cudaSuccess)
        return fail(c, KMC_ENOMEM, "partition output buffer");
    (void)parts;
    return KMC_OK;
}

static kmc_status check_partition_args(kmc_ctx* c, int parts, int granule, const int64_t* bounds) {
    if (!bounds) return fail(c, KMC_EINVAL, "NULL bounds");
    const long long M = strip_count(c);
    if (parts < 1 || parts > 4096) return fail(c, KMC_EINVAL, "parts must be in [1, 4096]");
    if (granule < 1 || M % granule || M < (long long)parts * granule)
        return fail(c, KMC_EINVAL, "need strips (%lld) a multiple of granule and >= parts*granule", M);
    return KMC_OK;
}

// shared tail: cdf kernel on c's strip buffer, results to the host
static kmc_status finish_partition(kmc_ctx* c, int parts, int granule, int64_t* bounds, uint64_t* strip_load,
                                   double* imb) {
    const long long M = strip_count(c);
    CUDA_TRY(c, launch_cdf_partition(c->strips, c->strips + M, M, parts, granule, c->wl_out, c->stream));
    CUDA_TRY(c, cudaMemcpyAsync(bounds, c->wl_out, (size_t)(parts + 1) * 8, cudaMemcpyDeviceToHost, c->stream));
    double tmp[2];
    CUDA_TRY(c, cudaMemcpyAsync(tmp, c->wl_out + parts + 1, 16, cudaMemcpyDeviceToHost, c->stream));
    if (strip_load) CUDA_TRY(c, cudaMemcpyAsync(strip_load, c->strips, (size_t)M * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (imb) { imb[0] = tmp[0]; imb[1] = tmp[1]; }
    return KMC_OK;
}

kmc_status kmc_workload_mark(kmc_ctx* c) {
    if (!c) return KMC_EINVAL;
    CUDA_TRY(c, cudaSetDevice(c->device));
    const size_t owned = (size_t)c->g.My_local * c->g.R * c->g.Mx;
    CUDA_TRY(c, cudaMemcpyAsync(c->wmark, c->wev, owned * 4, cudaMemcpyDeviceToDevice, c->stream));
    return KMC_OK;
}

kmc_status kmc_workload_partition(kmc_ctx* c, int32_t parts, int32_t granule, int64_t* bounds, uint64_t* strip_load,
                                  double* imbalance) {
    if (!c) return KMC_EINVAL;
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: use kmc_vgroup_workload_partition");
    kmc_status st = check_partition_args(c, parts, granule, bounds);
    if (st != KMC_OK) return st;
    CUDA_TRY(c, cudaSetDevice(c->device));
    st = ensure_strips(c, parts);
    if (st != KMC_OK) return st;
    const long long M = strip_count(c);
    CUDA_TRY(c, cudaMemsetAsync(c->strips, 0, (size_t)M * 8, c->stream));
    CUDA_TRY(c, launch_strip_loads(c->g, c->wev, c->wmark, c->strips, c->stream));
    if (c->world > 1 && c->comm)   // every rank gets the global strip loads, then the same bounds
        NCCL_TRY(c, g_nccl.AllReduce(c->strips, c->strips, (size_t)M, ncclUint64, ncclSum, c->comm, c->stream));
    return finish_partition(c, parts, granule, bounds, strip_load, imbalance);
}

kmc_status kmc_vgroup_workload_partition(kmc_ctx** cs, int32_t world, int32_t parts, int32_t granule, int64_t* bounds,
                                         uint64_t* strip_load, double* imbalance) {
    if (!cs || world < 2) return KMC_EINVAL;
    kmc_ctx* c0 = cs[0];
    kmc_status st = check_partition_args(c0, parts, granule, bounds);
    if (st != KMC_OK) return st;
    CUDA_TRY(c0, cudaSetDevice(c0->device));
    st = ensure_strips(c0, parts);
    if (st != KMC_OK) return st;
    const long long M = strip_count(c0);
    CUDA_TRY(c0, cudaMemsetAsync(c0->strips, 0, (size_t)M * 8, c0->stream));
    for (int r = 0; r < world; ++r)   // one device, one stream: every rank adds into rank 0's strips
        CUDA_TRY(c0, launch_strip_loads(cs[r]->g, cs[r]->wev, cs[r]->wmark, c0->strips, c0->stream));
    return finish_partition(c0, parts, granule, bounds, strip_load, imbalance);
}

kmc_status kmc_vgroup_create(const kmc_geometry* geom, const kmc_model* model, int32_t world, int32_t device,
                             void* stream, kmc_ctx** out) {
    return kmc_vgroup_create_bounds(geom, model, world, device, stream, nullptr, out);
}

kmc_status kmc_vgroup_create_bounds(const kmc_geometry* geom, const kmc_model* model, int32_t world, int32_t device,
                                    void* stream, const int64_t* row_bounds, kmc_ctx** out) {
    if (!geom || !model || !out || world < 2) return fail(nullptr, KMC_EINVAL, "vgroup needs world >= 2");
    if (geom->ndim != 2) return fail(nullptr, KMC_EINVAL, "vgroup: 2D lattices only (1D shards replicas)");
    for (int r = 0; r < world; ++r) out[r] = nullptr;
    // ONE stream for the whole group: the exchange copies of one rank read another rank's rows, so
    // everything must be ordered on a single stream.  If none is given the group creates it and the
    // last rank destroyed releases it (shared, reference counted).
    VgShared* sh = nullptr;
    if (!stream) {
        if (cudaSetDevice(device) != cudaSuccess) return fail(nullptr, KMC_ECUDA, "cudaSetDevice(%d)", device);
        sh = new VgShared();
        if (cudaStreamCreateWithFlags(&sh->stream, cudaStreamNonBlocking) != cudaSuccess) {
            delete sh;
            return fail(nullptr, KMC_ECUDA, "cudaStreamCreate failed");
        }
        stream = (void*)sh->stream;
    }
    for (int r = 0; r < world; ++r) {
        kmc_dist d{};
        d.rank = r; d.world = world; d.device = device; d.nccl_unique_id = nullptr; d.stream = stream;
        d.row_bounds = row_bounds;
        kmc_status st = create_ctx(geom, model, &d, true, &out[r]);
        if (st != KMC_OK) {
            // ranks 0..r-1 each hold a reference: the last kmc_destroy releases the shared stream
            // (r == 0: nobody took one, release it here); sh is not touched after that
            const bool unowned = sh && r == 0;
            for (int q = 0; q < r; ++q) { kmc_destroy(out[q]); out[q] = nullptr; }
            if (unowned) { cudaStreamDestroy(sh->stream); delete sh; }
            return st;
        }
        if (sh) { out[r]->vg_shared = sh; ++sh->refs; }
    }
    return KMC_OK;
}

kmc_status kmc_vgroup_set_fused(kmc_ctx** cs, int32_t world, int32_t enable) {
    if (!cs || world < 2) return KMC_EINVAL;
    for (int r = 0; r < world; ++r)
        if (!cs[r] || !cs[r]->vgroup || cs[r]->world != world || cs[r]->rank != r)
            return fail(cs[0], KMC_EINVAL, "vgroup: contexts must be ranks 0..world-1 of one kmc_vgroup_create");
    for (int r = 0; r < world; ++r) {
        kmc_ctx* c = cs[r];
        kmc_ctx* up = cs[c->rank_up];
        kmc_ctx* dn = cs[c->rank_down];
        c->fused = enable != 0;
        for (int p = 0; p < 2; ++p) {
            c->peer_up[p] = enable ? up->planes[p] : nullptr;
            c->peer_dn[p] = enable ? dn->planes[p] : nullptr;
        }
        c->peer_up_rows = up->g.My_local;
    }
    return KMC_OK;
}

kmc_status kmc_vgroup_sync(kmc_ctx** cs, int32_t world) {
    if (!cs || world < 2) return KMC_EINVAL;
    CUDA_TRY(cs[0], cudaSetDevice(cs[0]->device));
    return vgroup_forward(cs, world);
}

kmc_status kmc_vgroup_run(kmc_ctx** cs, int32_t world, double T, double dt, kmc_scheme scheme) {
    if (!cs || world < 2) return KMC_EINVAL;
    kmc_ctx* c0 = cs[0];
    for (int r = 0; r < world; ++r)
        if (!cs[r] || !cs[r]->vgroup || cs[r]->world != world || cs[r]->rank != r)
            return fail(c0, KMC_EINVAL, "vgroup: contexts must be ranks 0..world-1 of one kmc_vgroup_create");
    if (!(dt > 0.0) || !(T >= 0.0) || std::isinf(T)) return fail(c0, KMC_EINVAL, "need dt > 0 and finite T >= 0");
    if (scheme < KMC_LIE || scheme > KMC_RANDOM) return fail(c0, KMC_EINVAL, "unknown scheme %d", (int)scheme);
    CUDA_TRY(c0, cudaSetDevice(c0->device));
    bool truncated = false;
    const bool fused = c0->fused;
    if (fused) {   // ghost rows current once; afterwards the window kernels keep them current
        kmc_status st = vgroup_forward(cs, world);
        if (st != KMC_OK) return st;
    }
    for (double d : macro_durations(T, dt, &truncated)) {
        for (const auto& sd : macro_schedule(scheme, c0->C, d, c0->geom.seed, c0->window)) {
            kmc_status st = fused ? KMC_OK : vgroup_forward(cs, world);
            for (int r = 0; r < world && st == KMC_OK; ++r) st = launch_window(cs[r], sd.first, sd.second);
            if (st == KMC_OK && !fused) st = vgroup_reverse(cs, world);
            if (st != KMC_OK) return st;
        }
        for (int r = 0; r < world; ++r) {
            cs[r]->time += d;
            kmc_status sr = record_sample(cs[r]);
            if (sr != KMC_OK) return sr;
        }
    }
    return truncated ? KMC_WTRUNCATED : KMC_OK;
}

kmc_status kmc_vgroup_run_nested(kmc_ctx** cs, int32_t world, double T, double dt, int32_t n_inner,
                                 kmc_scheme outer, kmc_scheme inner, int32_t block) {
    if (!cs || world < 2) return KMC_EINVAL;
    kmc_ctx* c0 = cs[0];
    for (int r = 0; r < world; ++r)
        if (!cs[r] || !cs[r]->vgroup || cs[r]->world != world || cs[r]->rank != r)
            return fail(c0, KMC_EINVAL, "vgroup: contexts must be ranks 0..world-1 of one kmc_vgroup_create");
    kmc_status st = check_nested(c0, T, dt, n_inner, outer, inner, block);
    if (st != KMC_OK) return st;
    CUDA_TRY(c0, cudaSetDevice(c0->device));
    bool truncated = false;
    for (double d : macro_durations(T, dt, &truncated)) {
        for (const auto& of : outer_factors(outer, d)) {
            const Nest nest{of.first, block};
            st = vgroup_forward(cs, world);
            for (int k = 0; k < n_inner && st == KMC_OK; ++k)
                for (const auto& sd : macro_schedule(inner, c0->C, of.second / (double)n_inner, c0->geom.seed, c0->window)) {
                    for (int r = 0; r < world && st == KMC_OK; ++r) st = launch_window(cs[r], sd.first, sd.second, ~0ull, &nest);
                    if (st != KMC_OK) break;
                }
            if (st == KMC_OK) st = vgroup_reverse(cs, world);
            if (st != KMC_OK) return st;
        }
        for (int r = 0; r < world; ++r) {
            cs[r]->time += d;
            kmc_status sr = record_sample(cs[r]);
            if (sr != KMC_OK) return sr;
        }
    }
    return truncated ? KMC_WTRUNCATED : KMC_OK;
}

// a8 counters of the current state into out[KMC_OBS_WORDS] (device), stream-ordered: [0..35] the
// observables kernel's counters, [36] events (all ranks), [37] windows, [38] time (double bits)
static kmc_status enqueue_obs(kmc_ctx* c, unsigned long long* out) {
    kmc_status st = fused_quiesce(c);
    if (st == KMC_OK) st = exchange_forward(c);   // ghosts current for the +y bonds of the last owned row
    if (st != KMC_OK) return st;
    ObsArgs a{};
    a.acc = c->obs_acc;
    a.ev_total = c->ev_total;
    a.g = c->g;
    a.plane0 = c->planes[0];
    a.plane1 = c->planes[1];
    a.nplanes = c->nplanes;
    a.C = c->C;
    a.out = out;
    a.windows = c->window;
    a.time = c->time;
    CUDA_TRY(c, launch_observables(a, c->stream));
    if (c->world > 1 && c->comm)   // NCCL ranks: global sums (virtual ranks return local counts)
        NCCL_TRY(c, g_nccl.AllReduce(out, out, kObsCounters + 1, ncclUint64, ncclSum, c->comm, c->stream));
    return KMC_OK;
}

static void decode_obs(const kmc_ctx* c, const unsigned long long* h, kmc_obs* o) {
    memset(o, 0, sizeof *o);
    double t;
    memcpy(&t, &h[kObsCounters + 2], 8);
    o->time = t;
    o->windows = h[kObsCounters + 1];
    o->events = h[kObsCounters];
    long long total = 0;
    for (int s = 0; s < 4; ++s) { o->n_state[s] = (int64_t)h[s]; total += (long long)h[s]; }
    for (int col = 0; col < 4; ++col)
        for (int s = 0; s < 4; ++s) o->n_state_by_colour[col][s] = (int64_t)h[4 + col * 4 + s];
    for (int a2 = 0; a2 < 4; ++a2)
        for (int b = a2; b < 4; ++b) {
            int64_t v = (int64_t)h[20 + a2 * 4 + b];
            if (b != a2) v += (int64_t)h[20 + b * 4 + a2];
            o->nn_pairs[a2][b] = o->nn_pairs[b][a2] = v;
        }
    for (int s = 0; s < 4; ++s) o->coverage[s] = total ? (double)o->n_state[s] / (double)total : 0.0;
    o->energy = -c->model.K * (double)o->nn_pairs[1][1] + c->model.h * (double)o->n_state[1];   // R24
}

kmc_status kmc_observables(kmc_ctx* c, kmc_obs* o, uint32_t* per_cell) {
    if (!c || !o) return fail(c, KMC_EINVAL, "NULL argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    // one rank: the kernel's last block writes the counters straight into mapped pinned memory; NCCL
    // ranks all-reduce a device buffer first, then copy
    const bool mapped = !c->comm;
    kmc_status st = enqueue_obs(c, mapped ? c->d_hobs : c->obs_buf);
    if (st != KMC_OK) return st;
    if (!mapped) CUDA_TRY(c, launch_copy_words(c->d_hobs, c->obs_buf, KMC_OBS_WORDS, c->stream));   // no copy engine
    if (c->fused_ipc) CUDA_TRY(c, cudaMemcpyAsync(c->h_flag, c->flags + 2, 8, cudaMemcpyDeviceToHost, c->stream));
    std::vector<uint32_t> wl;
    const long long owned = (long long)c->g.My_local * c->g.R * c->g.Mx;
    if (per_cell) {
        wl.resize((size_t)owned);
        CUDA_TRY(c, cudaMemcpyAsync(wl.data(), c->wev, (size_t)owned * 4, cudaMemcpyDeviceToHost, c->stream));
    }
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    if (c->fused_ipc && *c->h_flag) return fail(c, KMC_ECUDA, "fused exchange: a neighbour flag wait timed out (results void)");
    decode_obs(c, c->h_obs, o);
    if (per_cell) {   // device order [cy][r][cx] -> [r][cy][cx]
        const int R = c->g.R, My = c->g.My_local, Mx = c->g.Mx;
        for (int cy = 0; cy < My; ++cy)
            for (int r = 0; r < R; ++r)
                memcpy(per_cell + ((size_t)r * My + cy) * Mx, wl.data() + ((size_t)cy * R + r) * Mx, (size_t)Mx * 4);
    }
    return KMC_OK;
}

kmc_status kmc_device_errors(kmc_ctx* c, int32_t* bad_spins, int32_t* wait_timeouts) {
    if (!c) return KMC_EINVAL;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    unsigned int e = 0;
    unsigned long long to = 0;
    CUDA_TRY(c, cudaMemcpy(&e, c->err_flag, 4, cudaMemcpyDeviceToHost));
    if (c->fused_ipc) CUDA_TRY(c, cudaMemcpy(&to, c->flags + 2, 8, cudaMemcpyDeviceToHost));
    if (bad_spins) *bad_spins = e ? 1 : 0;
    if (wait_timeouts) *wait_timeouts = to ? 1 : 0;
    return KMC_OK;
}

kmc_status kmc_vgroup_observables(kmc_ctx** cs, int32_t world, kmc_obs* o) {
    if (!cs || world < 2 || !o) return KMC_EINVAL;
    kmc_ctx* c0 = cs[0];
    for (int r = 0; r < world; ++r)
        if (!cs[r] || !cs[r]->vgroup || cs[r]->world != world || cs[r]->rank != r)
            return fail(c0, KMC_EINVAL, "vgroup: contexts must be ranks 0..world-1 of one kmc_vgroup_create");
    CUDA_TRY(c0, cudaSetDevice(c0->device));
    kmc_status st = vgroup_forward(cs, world);        // ghost rows current for the +y bonds
    for (int r = 0; r < world && st == KMC_OK; ++r) st = enqueue_obs(cs[r], cs[r]->obs_buf);
    if (st != KMC_OK) return st;
    std::vector<unsigned long long> h((size_t)world * KMC_OBS_WORDS);
    for (int r = 0; r < world; ++r)
        CUDA_TRY(c0, cudaMemcpyAsync(h.data() + (size_t)r * KMC_OBS_WORDS, cs[r]->obs_buf, KMC_OBS_WORDS * 8,
                                     cudaMemcpyDeviceToHost, c0->stream));
    CUDA_TRY(c0, cudaStreamSynchronize(c0->stream));
    // the group sum of the integer counters and event totals (words 0..36); windows and time are
    // the same on every rank (lockstep); then the same decode as kmc_observables (R24 energy)
    for (int r = 1; r < world; ++r)
        for (int w = 0; w <= kObsCounters; ++w) h[(size_t)w] += h[(size_t)r * KMC_OBS_WORDS + w];
    decode_obs(c0, h.data(), o);
    return KMC_OK;
}

kmc_status kmc_observables_device(kmc_ctx* c, uint64_t* dev_counters) {
    if (!c || !dev_counters) return fail(c, KMC_EINVAL, "NULL argument");
    CUDA_TRY(c, cudaSetDevice(c->device));
    if (c->comm) {   // NCCL ranks all-reduce a device buffer; host destinations get it by a copy kernel
        cudaPointerAttributes at{};
        if (cudaPointerGetAttributes(&at, dev_counters) != cudaSuccess) {
            cudaGetLastError();
            return fail(c, KMC_EINVAL, "dev_counters is neither device nor pinned host memory");
        }
        if (at.type != cudaMemoryTypeDevice) {
            kmc_status st = enqueue_obs(c, c->obs_buf);
            if (st != KMC_OK) return st;
            CUDA_TRY(c, launch_copy_words(reinterpret_cast<unsigned long long*>(dev_counters), c->obs_buf,
                                          KMC_OBS_WORDS, c->stream));
            return KMC_OK;
        }
    }
    return enqueue_obs(c, reinterpret_cast<unsigned long long*>(dev_counters));
}

kmc_status kmc_obs_decode(const kmc_ctx* c, const uint64_t* counters, kmc_obs* out) {
    if (!c || !counters || !out) return KMC_EINVAL;
    decode_obs(c, reinterpret_cast<const unsigned long long*>(counters), out);
    return KMC_OK;
}

kmc_status kmc_correlation(kmc_ctx* c, int32_t rmax, int32_t state, int64_t* out_x, int64_t* out_y) {
    if (!c || !out_x || !out_y) return fail(c, KMC_EINVAL, "NULL argument");
    if (state < 0 || state >= c->nstates) return fail(c, KMC_EINVAL, "state %d out of range", state);
    const long long W = c->W, H = c->g.ndim == 2 ? (long long)c->geom.dims[0] : 1;   // global extents
    if (rmax < 0 || rmax > kMaxCorrR || rmax >= W || (c->g.ndim == 2 && rmax >= H))
        return fail(c, KMC_EINVAL, "rmax %d out of range (< lattice extent, <= %d)", rmax, kMaxCorrR);
    const bool do_y = c->g.ndim == 2;
    if (do_y && c->g.ghost && rmax > c->g.qy)
        return fail(c, KMC_EINVAL, "multi-rank y correlation needs rmax <= q_y (one ghost cell row)");
    CUDA_TRY(c, cudaSetDevice(c->device));
    kmc_status st = fused_quiesce(c);
    if (st == KMC_OK) st = exchange_forward(c);
    if (st != KMC_OK) return st;
    const int R1 = rmax + 1;
    unsigned long long* d = nullptr;
    CUDA_TRY(c, cudaMallocAsync((void**)&d, (size_t)2 * R1 * 8, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(d, 0, (size_t)2 * R1 * 8, c->stream));
    CorrArgs a{};
    a.g = c->g;
    a.plane0 = c->planes[0];
    a.plane1 = c->planes[1];
    a.nplanes = c->nplanes;
    a.state = state;
    a.rmax = rmax;
    a.do_y = do_y ? 1 : 0;
    a.out = d;
    CUDA_TRY(c, launch_correlation(a, c->stream));
    if (c->world > 1 && c->comm)
        NCCL_TRY(c, g_nccl.AllReduce(d, d, (size_t)2 * R1, ncclUint64, ncclSum, c->comm, c->stream));
    std::vector<unsigned long long> h((size_t)2 * R1);
    CUDA_TRY(c, cudaMemcpyAsync(h.data(), d, (size_t)2 * R1 * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaFreeAsync(d, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    for (int r = 0; r < R1; ++r) {
        out_x[r] = (int64_t)h[r];
        out_y[r] = (int64_t)h[R1 + r];
    }
    return KMC_OK;
}

// ---- f1: the coverage process (R30; Figs. path1D / autocorr1D / pdf2d / dynamics2d) ----
static long long sites_per_replica(const kmc_ctx* c) {
    return c->geom.ndim == 1 ? (long long)c->geom.dims[0] : (long long)c->geom.dims[0] * c->geom.dims[1];
}

kmc_status kmc_record_coverage(kmc_ctx* c, int32_t state, int64_t capacity) {
    if (!c) return KMC_EINVAL;
    if (capacity < 0) return fail(c, KMC_EINVAL, "capacity must be >= 0");
    if (capacity > 0 && (state < 0 || state >= c->nstates)) return fail(c, KMC_EINVAL, "state %d out of range", state);
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));          // no window may still append to the old buffer
    cudaFree(c->series);
    c->series = nullptr;
    c->series_cap = c->series_n = 0;
    if (capacity == 0) return KMC_OK;
    if (cudaMalloc((void**)&c->series, (size_t)capacity * c->g.R * 8) != cudaSuccess)
        return fail(c, KMC_ENOMEM, "coverage series buffer (%lld samples x %d replicas)", (long long)capacity, c->g.R);
    c->series_cap = capacity;
    c->series_state = state;
    return record_sample(c);                                 // sample 0: the current state
}

// the series with complete per-replica counts: 2D slabs over NCCL ranks hold partial row sums
static kmc_status full_series(kmc_ctx* c, unsigned long long** out, bool* owned) {
    *out = c->series;
    *owned = false;
    if (c->geom.ndim == 2 && c->world > 1 && c->comm) {
        const size_t n = (size_t)c->series_n * c->g.R;
        unsigned long long* t = nullptr;
        CUDA_TRY(c, cudaMallocAsync((void**)&t, n * 8 + 8, c->stream));
        NCCL_TRY(c, g_nccl.AllReduce(c->series, t, n, ncclUint64, ncclSum, c->comm, c->stream));
        *out = t;
        *owned = true;
    }
    return KMC_OK;
}

kmc_status kmc_coverage_series(kmc_ctx* c, int64_t* out, int64_t max_samples, int64_t* n_samples) {
    if (!c) return KMC_EINVAL;
    if (n_samples) *n_samples = c->series_n;
    if (!out || max_samples <= 0 || c->series_n == 0) return KMC_OK;
    CUDA_TRY(c, cudaSetDevice(c->device));
    unsigned long long* ser = nullptr;
    bool owned = false;
    kmc_status st = full_series(c, &ser, &owned);
    if (st != KMC_OK) return st;
    const long long n = std::min<long long>(max_samples, c->series_n);
    CUDA_TRY(c, cudaMemcpyAsync(out, ser, (size_t)n * c->g.R * 8, cudaMemcpyDeviceToHost, c->stream));
    if (owned) CUDA_TRY(c, cudaFreeAsync(ser, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    return KMC_OK;
}

kmc_status kmc_coverage_stats(kmc_ctx* c, int64_t first, int32_t max_lag, double* acf, double* moments, int32_t bins,
                              int64_t* hist) {
    if (!c) return KMC_EINVAL;
    if (c->vgroup) return fail(c, KMC_ESTATE, "virtual-rank context: counts are per slab (use kmc_coverage_series)");
    const long long n = c->series_n, nsite = sites_per_replica(c);
    if (first < 0 || first >= n) return fail(c, KMC_EINVAL, "first %lld outside the %lld recorded samples", (long long)first, n);
    if (max_lag < 0 || max_lag >= n - first) return fail(c, KMC_EINVAL, "max_lag %d must be < samples - first", max_lag);
    if (hist && (bins < 1 || bins > nsite + 1 || (double)(nsite + 1) * bins >= 9.2e18))
        return fail(c, KMC_EINVAL, "bins must be in [1, sites per replica + 1]");
    CUDA_TRY(c, cudaSetDevice(c->device));
    unsigned long long* ser = nullptr;
    bool owned = false;
    kmc_status st = full_series(c, &ser, &owned);
    if (st != KMC_OK) return st;
    const bool split = c->geom.ndim == 1 && c->world > 1 && c->comm;   // 1D: replicas sharded over ranks
    const long long M = split ? (long long)c->geom.replicas : (long long)c->g.R;
    const long long np = n - first;
    unsigned long long* d = nullptr;                         // [1 total][max_lag+1 acov][bins hist]
    const size_t nb = (size_t)(hist ? bins : 0);
    CUDA_TRY(c, cudaMallocAsync((void**)&d, (size_t)(2 + max_lag + nb) * 8, c->stream));
    CUDA_TRY(c, cudaMemsetAsync(d, 0, (size_t)(2 + max_lag + nb) * 8, c->stream));
    CUDA_TRY(c, launch_series_total(ser, first, n, c->g.R, d, c->stream));
    if (split) NCCL_TRY(c, g_nccl.AllReduce(d, d, 1, ncclUint64, ncclSum, c->comm, c->stream));
    unsigned long long tot = 0;
    CUDA_TRY(c, cudaMemcpyAsync(&tot, d, 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const double mean = (double)tot / ((double)nsite * (double)np * (double)M);
    double* dacov = reinterpret_cast<double*>(d + 1);
    unsigned long long* dhist = d + 2 + max_lag;
    CUDA_TRY(c, launch_series_acov(ser, first, n, c->g.R, max_lag, (double)nsite, mean, dacov, c->stream));
    if (split) NCCL_TRY(c, g_nccl.AllReduce(dacov, dacov, (size_t)max_lag + 1, ncclFloat64, ncclSum, c->comm, c->stream));
    if (hist) {
        CUDA_TRY(c, launch_series_hist(ser, first, n, c->g.R, nsite, bins, dhist, c->stream));
        if (split) NCCL_TRY(c, g_nccl.AllReduce(dhist, dhist, nb, ncclUint64, ncclSum, c->comm, c->stream));
    }
    std::vector<double> hacov((size_t)max_lag + 1);
    CUDA_TRY(c, cudaMemcpyAsync(hacov.data(), dacov, hacov.size() * 8, cudaMemcpyDeviceToHost, c->stream));
    if (hist) CUDA_TRY(c, cudaMemcpyAsync(hist, dhist, nb * 8, cudaMemcpyDeviceToHost, c->stream));
    CUDA_TRY(c, cudaFreeAsync(d, c->stream));
    if (owned) CUDA_TRY(c, cudaFreeAsync(ser, c->stream));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    const double g0 = hacov[0] / ((double)np * (double)M);
    if (moments) { moments[0] = mean; moments[1] = g0; }
    if (acf)
        for (int l = 0; l <= max_lag; ++l) {
            const double gl = hacov[(size_t)l] / ((double)(np - l) * (double)M);
            acf[l] = g0 > 0.0 ? gl / g0 : 0.0;
        }
    return KMC_OK;
}

kmc_status kmc_get_state(const kmc_ctx* c, uint64_t* windows, double* time) {
    if (!c) return KMC_EINVAL;
    if (windows) *windows = c->window;
    if (time) *time = c->time;
    return KMC_OK;
}

kmc_status kmc_set_state(kmc_ctx* c, uint64_t windows, double time) {
    if (!c) return KMC_EINVAL;
    // the window kernel's chunk counters alternate with the window parity (window w claims from
    // slot w & 1 and zeroes the other); an arbitrary new counter may repeat the last parity
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaMemsetAsync(c->queue, 0, 2 * sizeof(unsigned int), c->stream));
    c->window = windows;
    c->time = time;
    return KMC_OK;
}

kmc_status kmc_rate_table(const kmc_ctx* c, int32_t* n, int32_t* type, int32_t* dir, int32_t* kappa,
                          double* rate, uint64_t* rate_u64, int32_t* F) {
    if (!c) return KMC_EINVAL;
    if (n) *n = c->nclass;
    if (F) *F = c->F;
    for (int i = 0; i < c->nclass; ++i) {
        if (type) type[i] = c->ctype[i];
        if (dir) dir[i] = c->cdir[i];
        if (kappa) kappa[i] = c->ckappa[i];
        if (rate) rate[i] = c->crate[i];
        if (rate_u64) rate_u64[i] = c->crate_u64[i];
    }
    return KMC_OK;
}

kmc_status kmc_set_kernel(kmc_ctx* c, int32_t mode) {
    if (!c) return KMC_EINVAL;
    if (mode < KMC_KERNEL_AUTO || mode > KMC_KERNEL_GROUP32) return fail(c, KMC_EINVAL, "unknown kernel mode %d", mode);
    c->kernel_mode = mode;
    return KMC_OK;
}

kmc_status kmc_enable_timing(kmc_ctx* c, int32_t enable) {
    if (!c) return KMC_EINVAL;
    c->timing = enable != 0;
    return KMC_OK;
}

kmc_status kmc_timing(kmc_ctx* c, double* kernel_ms, int64_t* launches, int32_t reset) {
    if (!c) return KMC_EINVAL;
    CUDA_TRY(c, cudaSetDevice(c->device));
    CUDA_TRY(c, cudaStreamSynchronize(c->stream));
    double tot = 0.0;
    for (size_t i = 0; i < c->tev_used; ++i) {
        float ms = 0.f;
        CUDA_TRY(c, cudaEventElapsedTime(&ms, c->tev[i].first, c->tev[i].second));
        tot += ms;
    }
    if (kernel_ms) *kernel_ms = tot;
    if (launches) *launches = (int64_t)c->tev_used;
    if (reset) c->tev_used = 0;
    return KMC_OK;
}

}  // extern "C"
