// kmc_tile.cu -- shared-memory tile variant of the window kernel (2D spin-flip models).
//
// One CTA owns a TY x TX tile of cells.  It stages the tile plus its one-cell halo ring
// ((TY+2) x (TX+2) bit-board words, periodic wrap or ghost rows) into shared memory with
// coalesced row loads, then its lanes run the tile's active cells of the colour from a CTA-level
// queue (warp-aggregated shared-memory atomic), reading each cell's closure from shared memory
// instead of five scattered global loads.  Spin-flip events write only inside their own cell, so
// the staged halo words stay valid for the whole window and each finished cell is written back
// with one global store.  This removes the per-cell global-load latency that dominates when a
// window holds few events per cell (small dt, the HBM-bound end of SURVEY §8(d)); the event step
// itself is the same function as the lane-queue kernel's (kmc_device.cuh), so results are
// bit-identical.
#include "kmc_device.cuh"

#include <cstdint>

namespace kmc {

template <int TY, int TX, bool MH>
__global__ void __launch_bounds__(256, 3)
tile_kernel_adsdes2d(const SubstepArgs a, const int tiles_x) {
    constexpr int SW = TX + 2;                       // smem row stride (words)
    __shared__ uint64_t T[(TY + 2) * SW];
    __shared__ double2 s_logt[kLogTab];
    __shared__ uint8_t s_sel8[kSel8];
    __shared__ uint32_t s_next;
    const Geo& g = a.g;
    const unsigned FULL = 0xffffffffu;
    const int tid = threadIdx.x, lane = tid & 31;

    // tile coordinates: x fastest, then replica, then tile row
    const int bx = blockIdx.x % tiles_x;
    const int rest = blockIdx.x / tiles_x;
    const int r = rest % g.R;
    const int by = rest / g.R;
    const int x0 = bx * TX, y0 = by * TY;
    const int w = min(TX, g.Mx - x0), h = min(TY, g.My_local - y0);     // both even (R7 + launch)
    const uint32_t rowlen = (uint32_t)g.R * g.Mx;
    const uint32_t rbase = (uint32_t)r * g.Mx;

    for (int i = tid; i < kLogTab; i += blockDim.x) s_logt[i] = a.logtab[i];
    init_sel8(s_sel8);
    if (tid == 0) s_next = blockDim.x;
    // a3: the tile and its halo ring, row by row (coalesced), periodic wrap / ghost rows
    const int hw = w + 2, nload = (h + 2) * hw;
    for (int i = tid; i < nload; i += blockDim.x) {
        const int ly = i / hw, lx = i - ly * hw;
        int cy = y0 + ly - 1, cx = x0 + lx - 1;
        cx = cx < 0 ? cx + g.Mx : (cx >= g.Mx ? cx - g.Mx : cx);
        int sy = cy + g.ghost;
        if (!g.ghost) sy = sy < 0 ? sy + g.My_local : (sy >= g.My_local ? sy - g.My_local : sy);
        T[ly * SW + lx] = a.plane0[(uint32_t)sy * rowlen + rbase + (uint32_t)cx];
    }
    __syncthreads();

    // active cells of the colour in this tile, numbered row-major
    const int gy0 = g.row_offset + y0;
    const uint32_t half = (uint32_t)w >> 1;
    const uint32_t nact = (a.C == 2) ? (uint32_t)h * half : (uint32_t)(h >> 1) * half;
    const double inv_half = 1.0 / (double)half;
    auto cell_of = [&](uint32_t t, int& lr, int& lc) {
        uint32_t i, j;
        fast_divmod(t, half, inv_half, i, j);
        if (a.C == 2) { lr = (int)i; lc = 2 * (int)j + ((a.colour + gy0 + lr) & 1); }
        else { lr = 2 * (int)i + (a.colour >> 1); lc = 2 * (int)j + (a.colour & 1); }
    };

    uint32_t t = tid;
    bool have = t < nact;
    int lr = 0, lc = 0;
    uint32_t gid32 = 0, k = 0;
    double tclock = 0.0;
    uint64_t P[1] = {}, hb[1][4] = {};
    unsigned long long evsum = 0;
    auto load = [&]() {
        cell_of(t, lr, lc);
        const int c0 = (lr + 1) * SW + (lc + 1);
        P[0] = T[c0];
        halo_from_words<MH>(g, T[c0 - 1], T[c0 + 1], T[c0 - SW], T[c0 + SW], hb[0], true);
        gid32 = (uint32_t)((unsigned long long)(g.rep_offset + r) * (unsigned long long)g.M_global +
                           (unsigned long long)(gy0 + lr) * g.Mx + (x0 + lc));
        k = 0;
        tclock = 0.0;
    };
    if (have) load();
    if (!__any_sync(FULL, have)) return;                          // warp beyond the tile's cells
    for (;;) {
        const bool fin = event_step<0, 2, MH>(a, P, hb, k, tclock, gid32, have, s_logt, s_sel8);
        const unsigned fm = __ballot_sync(FULL, fin);
        if (fm) {                                                   // warp-uniform
            uint32_t base = 0;
            if (lane == 0) base = atomicAdd(&s_next, (uint32_t)__popc(fm));
            base = __shfl_sync(FULL, base, 0);
            if (fin) {
                if (k) {   // a6: write the cell back once, count its events
                    const uint32_t gi = (uint32_t)(y0 + lr + g.ghost) * rowlen + rbase + (uint32_t)(x0 + lc);
                    a.plane0[gi] = P[0];
                    atomicAdd(&a.wev[(uint32_t)(y0 + lr) * rowlen + rbase + (uint32_t)(x0 + lc)], k);   // RED
                    evsum += k;
                }
                t = base + __popc(fm & ((1u << lane) - 1u));
                have = t < nact;
                if (have) load();
            }
            if (!__any_sync(FULL, have)) break;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evsum += __shfl_xor_sync(FULL, evsum, o);
    if (lane == 0 && evsum) atomicAdd(a.ev_total, evsum);
}

// Tile kernel for 2D spin-flip windows; returns cudaErrorNotSupported when the geometry does not
// fit it (the caller then uses the lane-queue kernel).
cudaError_t launch_substep_tile(const SubstepArgs& a, cudaStream_t s) {
    const Geo& g = a.g;
    if (g.ndim != 2) return cudaErrorNotSupported;
    constexpr int TY = 32, TX = 64;
    const int tiles_x = (g.Mx + TX - 1) / TX;
    const int tiles_y = (g.My_local + TY - 1) / TY;
    const long long nb = (long long)tiles_x * tiles_y * g.R;
    if (nb <= 0 || nb > 0x7fffffffLL) return cudaErrorNotSupported;
    if (g.qx >= 2 && g.qy >= 2) tile_kernel_adsdes2d<TY, TX, true><<<(unsigned)nb, 256, 0, s>>>(a, tiles_x);
    else tile_kernel_adsdes2d<TY, TX, false><<<(unsigned)nb, 256, 0, s>>>(a, tiles_x);
    return cudaGetLastError();
}

}  // namespace kmc
