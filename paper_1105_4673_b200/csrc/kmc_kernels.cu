// kmc_kernels.cu -- sm_100a kernels of the fractional-step KMC hot path.
//
// substep_kernel: one window e^{D L^c} of eq.(exact).
//   ONE LANE OWNS ONE COARSE CELL.  The cell and its one-site halo live in registers as
//   64-bit bitboards (bit-packed cell-major layout, kmc_internal.h); per event the lane
//     1. derives every slot class's member mask by bit-sliced neighbour counting
//        (the class is the rate-table index of eq.(Arrhenius) P:963-968 / Table COrates),
//     2. lambda = sum_c popc(mask_c) * rate_c   (eq.(totalrate), exact u64)
//     3. draws Philox4x32-10(k, gid, window) and the exponential clock tau = -ln U / lambda
//        (fdlibm log, IEEE RN ops only -- DESIGN.md §3), stops when t + tau >= D (R5),
//     4. picks class c with prob popc*rate/lambda and a uniform member site of c
//        (eq.(skeleton)) with popc-based rank selection, and
//     5. applies the event as XORs on the planes (partner sites outside the cell go to
//        the halo boards, written back once per window with atomicXor of the delta).
//   No tensor cores: this is not a contraction.  See DESIGN.md §8 for why a lane (not a
//   warp) owns a cell: the per-event chain is serial, so 32 independent cells per warp
//   give 32x the issue efficiency of a warp-cooperative scan.
// observables_kernel (a8): integer counts, order-free.
// pack / unpack: uint8 site-major <-> bit-packed cell-major.
#include "kmc_internal.h"

#include <cstdint>
#include <cstdlib>

namespace kmc {

// ---------------------------------------------------------------------------------------------
// L0 arithmetic: Philox4x32-10 and the fdlibm log sequence.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0);
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// natural log on normal x in (0, 1]: x = 2^e m, m in [sqrt(2)/2, sqrt(2)),
// bucket j = round(128 m) - 91, r = fma(m, c_j, -1), log x = e ln2 + L_j + r + r^2 q(r) with q the
// Taylor polynomial of log1p to r^7.  Division-free and branch-free; every step one explicit
// round-to-nearest operation (__fma_rn / __dmul_rn / __dadd_rn) so the bits match the CPU oracle.
// ctab / ltab: the kLogTab-entry tables staged in shared memory.
__device__ __forceinline__ double log_spec(double x, const double* ctab, const double* ltab, const double* lc) {
    // lc = {1/7, -1/6, 1/5, 1/3, ln2_hi, ln2_lo} from the kernel parameters (constant bank operands:
    // full 64-bit FP64 constants would otherwise be rebuilt with uniform moves every event)
    const double ln2_hi = lc[4], ln2_lo = lc[5];
    const unsigned long long u = (unsigned long long)__double_as_longlong(x);
    const int e0 = (int)((u >> 52) & 0x7ff) - 1023;
    const unsigned long long mant = u & 0xFFFFFFFFFFFFFull;
    const bool hi = mant >= 0x6A09E667F3BCDull;                   // 1.mant >= sqrt(2): halve
    const int e = e0 + (hi ? 1 : 0);
    const int idx = hi ? 64 + (int)((mant + (1ull << 45)) >> 46) : 128 + (int)((mant + (1ull << 44)) >> 45);
    const double m = __longlong_as_double((long long)((hi ? 0x3FE0000000000000ull : 0x3FF0000000000000ull) | mant));
    const int j = idx - 91;
    const double r = __fma_rn(m, ctab[j], -1.0);
    double q = __fma_rn(r, lc[0], lc[1]);
    q = __fma_rn(r, q, lc[2]);
    q = __fma_rn(r, q, -0.25);
    q = __fma_rn(r, q, lc[3]);
    q = __fma_rn(r, q, -0.5);
    const double p = __fma_rn(__dmul_rn(r, r), q, r);
    const double dk = (double)e;
    double s = __dadd_rn(ltab[j], p);
    s = __fma_rn(dk, ln2_lo, s);
    return __fma_rn(dk, ln2_hi, s);
}

// q = n / d, rem = n % d for n < 2^32 via the FP64 reciprocal inv = RN(1/d): n*inv is within
// 2^-52 relative of n/d, so floor(n*inv) is floor(n/d) or, when n/d is an integer, possibly one
// less -- fixed by one compare.  ~7 instructions instead of a ~40-instruction integer division.
__device__ __forceinline__ void fast_divmod(uint32_t n, uint32_t d, double inv, uint32_t& q, uint32_t& rem) {
    q = __double2uint_rz(__dmul_rn(__uint2double_rn(n), inv));
    rem = n - q * d;
    if (rem >= d) { ++q; rem -= d; }
}

// position of the k-th (0-based) set bit of a 64-bit word (k < popc(m))
__device__ __forceinline__ int select_bit64(uint64_t m, uint32_t k) {
    uint32_t w = (uint32_t)m;
    int pos = 0;
    const uint32_t pl = __popc(w);
    if (k >= pl) { k -= pl; w = (uint32_t)(m >> 32); pos = 32; }
    uint32_t c = __popc(w & 0xFFFFu);
    if (k >= c) { k -= c; w >>= 16; pos += 16; }
    c = __popc(w & 0xFFu);
    if (k >= c) { k -= c; w >>= 8; pos += 8; }
    c = __popc(w & 0xFu);
    if (k >= c) { k -= c; w >>= 4; pos += 4; }
    c = __popc(w & 0x3u);
    if (k >= c) { k -= c; w >>= 2; pos += 2; }
    c = w & 1u;
    if (k >= c) { pos += 1; }
    return pos;
}

// ---------------------------------------------------------------------------------------------
// Models: class masks in canonical order and per-class XOR descriptors.
// desc bits: 0 anchor toggles plane0, 1 anchor toggles plane1, 2 partner toggles plane0,
//            3 partner toggles plane1, 4-5 direction, 6 has partner.
// Directions d: 0 = -x, 1 = +x, 2 = -y, 3 = +y.
// nb[p][d] = bitboard of plane p at the neighbour x+e_d of every cell site.
// ---------------------------------------------------------------------------------------------
constexpr int D_A0 = 1, D_A1 = 2, D_P0 = 4, D_P1 = 8, D_HASP = 64;
__host__ __device__ constexpr int dsh(int d) { return d << 4; }

// n == k masks from the z neighbour boards of plane 0 (bit-sliced adder)
template <int NDIM>
__device__ __forceinline__ void eq_counts(const uint64_t* nb, uint64_t* eq) {
    if (NDIM == 1) {
        eq[0] = ~(nb[0] | nb[1]);
        eq[1] = nb[0] ^ nb[1];
        eq[2] = nb[0] & nb[1];
    } else {
        const uint64_t s1 = nb[0] ^ nb[1], c1 = nb[0] & nb[1];
        const uint64_t s2 = nb[2] ^ nb[3], c2 = nb[2] & nb[3];
        const uint64_t b0 = s1 ^ s2, cr = s1 & s2;
        const uint64_t b1 = c1 ^ c2 ^ cr;
        const uint64_t b2 = (c1 & c2) | (cr & (c1 ^ c2));
        eq[0] = ~(b0 | b1 | b2);
        eq[1] = b0 & ~b1 & ~b2;
        eq[2] = ~b0 & b1 & ~b2;
        eq[3] = b0 & b1 & ~b2;
        eq[4] = b2;                                       // n = 4 (b2 set implies b0 = b1 = 0)
    }
}

template <int KIND, int NDIM> struct Model;

template <int NDIM> struct Model<0, NDIM> {                    // ADSDES
    static constexpr int Z = 2 * NDIM, NP = 1, NC = 2 + Z;
    __device__ static int desc(int) { return D_A0; }
    __device__ static void masks(const uint64_t* P, const uint64_t (*nb)[4], uint64_t valid, uint64_t* m) {
        uint64_t eq[Z + 1];
        eq_counts<NDIM>(nb[0], eq);
        m[0] = valid & ~P[0];
#pragma unroll
        for (int n = 0; n <= Z; ++n) m[1 + n] = P[0] & eq[n];
    }
};

template <int NDIM> struct Model<1, NDIM> {                    // ADSDES_DIFF
    static constexpr int Z = 2 * NDIM, NP = 1, NC = 2 + Z + Z * Z;
    __device__ static int desc(int c) {
        if (c < 2 + Z) return D_A0;
        const int d = (c - 2 - Z) / Z;
        return D_A0 | D_P0 | D_HASP | dsh(d);
    }
    __device__ static void masks(const uint64_t* P, const uint64_t (*nb)[4], uint64_t valid, uint64_t* m) {
        uint64_t eq[Z + 1];
        eq_counts<NDIM>(nb[0], eq);
        m[0] = valid & ~P[0];
#pragma unroll
        for (int n = 0; n <= Z; ++n) m[1 + n] = P[0] & eq[n];
#pragma unroll
        for (int d = 0; d < Z; ++d) {
            const uint64_t mover = P[0] & ~nb[0][d];
#pragma unroll
            for (int n = 0; n < Z; ++n) m[2 + Z + d * Z + n] = mover & eq[n];
        }
    }
};

template <int KIND, int NDIM> struct ZgbModel {                // ZGB (KIND 2) / ZGB_DIFF (KIND 3)
    static constexpr int Z = 2 * NDIM, NP = 2, NC = 1 + 3 * Z + (KIND == 3 ? Z : 0);
    __device__ static int desc(int c) {
        if (c == 0) return D_A0;                                   // CO adsorb
        const int g = (c - 1) / Z, d = (c - 1) % Z;
        if (g == 0) return D_A1 | D_P1 | D_HASP | dsh(d);          // O2 adsorb: x, y -> O
        if (g == 1) return D_A0 | D_P1 | D_HASP | dsh(d);          // CO(x) + O(y) -> vacant
        if (g == 2) return D_A1 | D_P0 | D_HASP | dsh(d);          // O(x) + CO(y) -> vacant
        return D_A0 | D_P0 | D_HASP | dsh(d);                      // CO hop x -> y
    }
    __device__ static void masks(const uint64_t* P, const uint64_t (*nb)[4], uint64_t valid, uint64_t* m) {
        const uint64_t vac = valid & ~(P[0] | P[1]);
        m[0] = vac;
#pragma unroll
        for (int d = 0; d < Z; ++d) {
            const uint64_t vnb = ~(nb[0][d] | nb[1][d]);
            m[1 + d] = vac & vnb;
            m[1 + Z + d] = P[0] & nb[1][d];
            m[1 + 2 * Z + d] = P[1] & nb[0][d];
            if (KIND == 3) m[1 + 3 * Z + d] = P[0] & vnb;
        }
    }
};
template <int NDIM> struct Model<2, NDIM> : ZgbModel<2, NDIM> {};
template <int NDIM> struct Model<3, NDIM> : ZgbModel<3, NDIM> {};

// ---------------------------------------------------------------------------------------------
// The window kernel.
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
    uint32_t iev;                     // index into the per-cell event counters
    uint32_t gid32;                   // global cell id (Philox counter word 1, R17)
};

// Active-cell number t -> cell location.  All indices fit 32 bits (kmc_create enforces < 2^32
// cells in total, and a plane holds at most that many words plus two ghost rows).
template <int NDIM>
__device__ __forceinline__ CellLoc locate(const SubstepArgs& a, uint32_t t) {
    const Geo& g = a.g;
    const uint32_t half = (uint32_t)g.Mx >> 1;
    uint32_t rest, j, rowsel, r;
    fast_divmod(t, half, a.inv_half, rest, j);
    if (g.R == 1) { rowsel = rest; r = 0; }
    else fast_divmod(rest, (uint32_t)g.R, a.inv_R, rowsel, r);
    uint32_t cy, cx;
    if (NDIM == 1) {
        cy = 0;
        cx = 2 * j + a.colour;
    } else if (a.C == 2) {
        cy = rowsel;
        cx = 2 * j + ((a.colour + g.row_offset + cy) & 1);
    } else {
        cy = 2 * rowsel + (a.colour >> 1);
        cx = 2 * j + (a.colour & 1);
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
    L.iC = base + cx;
    L.iW = base + cxW;
    L.iE = base + cxE;
    L.iN = (uint32_t)syN * rowlen + rbase + cx;
    L.iS = (uint32_t)syS * rowlen + rbase + cx;
    L.iev = cy * rowlen + rbase + cx;
    L.gid32 = (uint32_t)((unsigned long long)(g.rep_offset + r) * (unsigned long long)g.M_global +
                         (unsigned long long)gy * g.Mx + cx);
    return L;
}

template <int KIND, int NDIM, int BS, int MINB>
__global__ void __launch_bounds__(BS, MINB)
substep_kernel(const SubstepArgs a, const uint32_t nactive, const uint32_t chunk) {
    using M = Model<KIND, NDIM>;
    constexpr int NP = M::NP, NC = M::NC;
    const Geo& g = a.g;
    const unsigned FULL = 0xffffffffu;
    // log_spec tables -> shared memory (lanes index them by their own bucket)
    __shared__ double s_logc[kLogTab], s_logl[kLogTab];
    for (int i = threadIdx.x; i < kLogTab; i += blockDim.x) { s_logc[i] = a.log_c[i]; s_logl[i] = a.log_l[i]; }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long cbeg64 = (unsigned long long)warp * chunk;
    if (cbeg64 >= nactive) return;                                  // warp-uniform
    const uint32_t cbeg = (uint32_t)cbeg64;
    const uint32_t cend = (uint32_t)min(cbeg64 + chunk, (unsigned long long)nactive);
    const uint64_t notcol0 = g.notcol0, notcolL = g.notcolL;
    const uint64_t notrow0 = g.notrow0, notrowL = g.notrowL;
    uint64_t* planes[2] = {a.plane0, a.plane1};

    uint32_t next = cbeg + 32;                                      // warp-uniform queue head
    uint32_t ci = cbeg + lane;
    bool have = ci < cend;
    uint32_t gid32 = 0, k = 0;
    double tclock = 0.0;
    uint64_t P[NP], h[NP][4];
    unsigned long long evsum = 0;

    // a3: stage the closure (cell + one-site halo) of cell `ci` into registers
    auto load = [&](uint32_t c) {
        const CellLoc L = locate<NDIM>(a, c);
        gid32 = L.gid32;
        k = 0;
        tclock = 0.0;
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            const uint64_t* pl = planes[p];
            P[p] = pl[L.iC];
            h[p][0] = (pl[L.iW] >> (g.qx - 1)) & g.col0;           // sigma(x-1) seen by column 0
            h[p][1] = (pl[L.iE] << (g.qx - 1)) & g.colL;           // sigma(x+1) seen by column qx-1
            if (NDIM == 2) {
                h[p][2] = (pl[L.iN] >> g.shN) & g.row0;             // sigma(y-1) seen by row 0
                h[p][3] = (pl[L.iS] << g.shN) & g.rowL;             // sigma(y+1) seen by row qy-1
            } else {
                h[p][2] = h[p][3] = 0;
            }
        }
    };
    // a6: write the cell back once per window (+ halo deltas for hop / pair events)
    auto store = [&](uint32_t c) {
        if (k == 0) return;
        const CellLoc L = locate<NDIM>(a, c);
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            uint64_t* pl = planes[p];
            pl[L.iC] = P[p];
            if (KIND != 0) {
                // halo deltas.  Our halo bits of the neighbour words are written by no other cell
                // in this window (same-colour closures are disjoint, R6), so re-reading them gives
                // the window-start values; the XOR touches only those bits (order-free).
                const uint64_t dW = h[p][0] ^ ((pl[L.iW] >> (g.qx - 1)) & g.col0);
                const uint64_t dE = h[p][1] ^ ((pl[L.iE] << (g.qx - 1)) & g.colL);
                if (dW) atomicXor((unsigned long long*)&pl[L.iW], (unsigned long long)(dW << (g.qx - 1)));
                if (dE) atomicXor((unsigned long long*)&pl[L.iE], (unsigned long long)(dE >> (g.qx - 1)));
                if (NDIM == 2) {
                    const uint64_t dN = h[p][2] ^ ((pl[L.iN] >> g.shN) & g.row0);
                    const uint64_t dS = h[p][3] ^ ((pl[L.iS] << g.shN) & g.rowL);
                    if (dN) atomicXor((unsigned long long*)&pl[L.iN], (unsigned long long)(dN << g.shN));
                    if (dS) atomicXor((unsigned long long*)&pl[L.iS], (unsigned long long)(dS >> g.shN));
                }
            }
        }
        a.wev[L.iev] += k;
        evsum += k;
    };

    if (have) load(ci);
    // The event step is one branch-free basic block: lanes without a cell (queue exhausted) and
    // lanes whose window ended compute it too, with the update masked off (ab = 0), so the warp
    // never diverges inside the step and the scheduler can interleave its independent chains.
    for (;;) {
        // RNG and -ln U first: independent of lambda, so they overlap the mask chain (ILP)
        uint4 x = make_uint4(k, gid32, a.w_lo, a.w_hi_tag);
#pragma unroll
        for (int rd = 0; rd < 10; ++rd) {
            const uint32_t lo0 = 0xD2511F53u * x.x, hi0 = __umulhi(0xD2511F53u, x.x);
            const uint32_t lo1 = 0xCD9E8D57u * x.z, hi1 = __umulhi(0xCD9E8D57u, x.z);
            x = make_uint4(hi1 ^ x.y ^ a.rk0[rd], lo1, hi0 ^ x.w ^ a.rk1[rd], lo0);
        }
        const uint64_t j53 = ((uint64_t)x.x << 21) | (uint64_t)(x.y >> 11);
        const double U = __dmul_rn(__ull2double_rn(j53 + 1ull), 0x1p-53);
        const double E = -log_spec(U, s_logc, s_logl, a.lcoef);

        // a4/a5: class masks, counts and lambda (eq.(totalrate), exact u64)
        uint64_t nb[NP][4];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
            nb[p][0] = ((P[p] << 1) & notcol0) | h[p][0];
            nb[p][1] = ((P[p] >> 1) & notcolL) | h[p][1];
            if (NDIM == 2) {
                nb[p][2] = ((P[p] << g.qx) & g.valid) | h[p][2];
                nb[p][3] = (P[p] >> g.qx) | h[p][3];
            } else {
                nb[p][2] = nb[p][3] = 0;
            }
        }
        uint64_t m[NC];
        M::masks(P, nb, g.valid, m);
        uint32_t cnt[NC];
        uint64_t lam = 0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            cnt[c] = __popcll(m[c]);
            lam += (uint64_t)cnt[c] * a.rate[c];
        }
        const double lamd = __dmul_rn(__ull2double_rn(lam), a.inv_scale);
        const double tau = __ddiv_rn(E, lamd);
        const double tn = __dadd_rn(tclock, tau);
        // accept unless quiescent (lambda = 0) or past the window end (R5: pending event discarded)
        const bool accept = have && lam != 0 && tn < a.D;
        const bool fin = have && !accept;
        tclock = accept ? tn : tclock;
        // eq.(skeleton): class = smallest c with prefix(c) > r, r = floor(x2 lambda / 2^32)
        const uint64_t rr = (uint64_t)x.z * (lam >> 32) + (uint64_t)__umulhi(x.z, (uint32_t)lam);
        uint64_t cum = 0, selm = m[NC - 1];
        uint32_t selc = cnt[NC - 1];
        int seld = M::desc(NC - 1);
        bool found = false;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            cum += (uint64_t)cnt[c] * a.rate[c];
            const bool hit = !found && cum > rr;
            selm = hit ? m[c] : selm;
            selc = hit ? cnt[c] : selc;
            seld = hit ? M::desc(c) : seld;
            found = found || hit;
        }
        // site: the kk-th member of the class in row-major order, kk = floor(x3 cnt / 2^32)
        const int s = select_bit64(selm, __umulhi(x.w, selc));
        const uint64_t ab = accept ? (1ull << s) : 0ull;
        if (seld & D_A0) P[0] ^= ab;
        if (NP > 1 && (seld & D_A1)) P[NP - 1] ^= ab;
        if (seld & D_HASP) {
            const int d = (seld >> 4) & 3;
            const uint64_t inner = d == 0 ? notcol0 : d == 1 ? notcolL : d == 2 ? notrow0 : notrowL;
            const uint64_t pb = d == 0 ? ab >> 1 : d == 1 ? ab << 1 : d == 2 ? ab >> g.qx : ab << g.qx;
            const bool in_cell = (ab & inner) != 0;
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const bool tog = (seld & (D_P0 << p)) != 0;
                P[p] ^= (tog && in_cell) ? pb : 0ull;
#pragma unroll
                for (int dd = 0; dd < 4; ++dd) h[p][dd] ^= (tog && !in_cell && dd == d) ? ab : 0ull;
            }
        }
        k += accept ? 1u : 0u;

        const unsigned fm = __ballot_sync(FULL, fin);
        if (fm) {                                                  // warp-uniform
            if (fin) {
                store(ci);
                ci = next + __popc(fm & ((1u << lane) - 1u));
                have = ci < cend;
                if (have) load(ci);
            }
            next += __popc(fm);
            if (!__any_sync(FULL, have)) break;
        }
    }
    // event total: warp-aggregated
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) evsum += __shfl_xor_sync(FULL, evsum, o);
    if (lane == 0 && evsum) atomicAdd(a.ev_total, evsum);
}

template <int KIND, int NDIM>
static cudaError_t launch_t(const SubstepArgs& a, long long nactive, cudaStream_t s) {
    if (nactive <= 0) return cudaSuccess;
    // launch shape (block size, min blocks per SM): env KMC_LB selects an experiment variant
    static const int lb = [] { const char* e = getenv("KMC_LB"); return e ? atoi(e) : 0; }();
    int bs = 256;
    if (KIND == 0 && (lb == 1 || lb == 2)) bs = 128;
    // cells per warp: 32 lanes x a few cells each, so a lane's tail idles for ~1/cpl of the window
    long long cpl = 8;
    while (cpl > 1 && (nactive + 32 * cpl - 1) / (32 * cpl) < 4 * 148 * 8) cpl >>= 1;   // keep >= ~4 waves
    const long long chunk = 32 * cpl;
    const long long nwarps = (nactive + chunk - 1) / chunk;
    const unsigned nb = (unsigned)((nwarps * 32 + bs - 1) / bs);
    const uint32_t na = (uint32_t)nactive, ch = (uint32_t)chunk;
    if constexpr (KIND == 0) {
        // spin flip default: <= 80 registers, 3 blocks of 256 (24 warps) per SM
        if (lb == 1) substep_kernel<KIND, NDIM, 128, 5><<<nb, 128, 0, s>>>(a, na, ch);        // <= 96 regs, 20 warps
        else if (lb == 2) substep_kernel<KIND, NDIM, 128, 4><<<nb, 128, 0, s>>>(a, na, ch);   // <= 128 regs, 16 warps
        else if (lb == 3) substep_kernel<KIND, NDIM, 256, 2><<<nb, 256, 0, s>>>(a, na, ch);   // <= 128 regs, 16 warps
        else substep_kernel<KIND, NDIM, 256, 3><<<nb, 256, 0, s>>>(a, na, ch);
    } else {
        substep_kernel<KIND, NDIM, 256, 2><<<nb, 256, 0, s>>>(a, na, ch);
    }
    return cudaGetLastError();
}

cudaError_t launch_substep(int kind, const SubstepArgs& a, long long nactive, cudaStream_t s) {
    const bool two = a.g.ndim == 2;
    switch (kind) {
    case 0: return two ? launch_t<0, 2>(a, nactive, s) : launch_t<0, 1>(a, nactive, s);
    case 1: return two ? launch_t<1, 2>(a, nactive, s) : launch_t<1, 1>(a, nactive, s);
    case 2: return two ? launch_t<2, 2>(a, nactive, s) : launch_t<2, 1>(a, nactive, s);
    case 3: return two ? launch_t<3, 2>(a, nactive, s) : launch_t<3, 1>(a, nactive, s);
    }
    return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------------------------
// a8: observables.  Counters (u64): [0..3] n_state, [4..19] by colour [c*4+s],
// [20..35] ordered nearest-neighbour bonds (x, x+e) for e in {+x, +y}: [20 + a*4 + b].
// ---------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(256) observables_kernel(const ObsArgs a) {
    const Geo& g = a.g;
    __shared__ unsigned long long sh[kObsCounters];
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    uint32_t acc[kObsCounters];
#pragma unroll
    for (int i = 0; i < kObsCounters; ++i) acc[i] = 0;
    const long long rowlen = (long long)g.R * g.Mx;
    const long long ncell = (long long)g.My_local * rowlen;
    for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < ncell;
         t += (long long)gridDim.x * blockDim.x) {
        const int cx = (int)(t % g.Mx);
        const long long rest = t / g.Mx;
        const int r = (int)(rest % g.R);
        const int cy = (int)(rest / g.R);
        const int sy = cy + g.ghost;
        int syS = sy + 1;
        if (!g.ghost && syS >= g.My_local) syS -= g.My_local;
        const int cxE = cx == g.Mx - 1 ? 0 : cx + 1;
        const long long iC = (long long)sy * rowlen + (long long)r * g.Mx + cx;
        const long long iE = (long long)sy * rowlen + (long long)r * g.Mx + cxE;
        const long long iS = (long long)syS * rowlen + (long long)r * g.Mx + cx;
        uint64_t A[3], Bx[3], By[3];
        const uint64_t notcolL = g.valid & ~g.colL;
        uint64_t occ = 0, occx = 0, occy = 0;
        for (int p = 0; p < a.nplanes; ++p) {
            const uint64_t* pl = p == 0 ? a.plane0 : a.plane1;
            const uint64_t P = pl[iC];
            A[1 + p] = P;
            Bx[1 + p] = ((P >> 1) & notcolL) | ((pl[iE] << (g.qx - 1)) & g.colL);
            By[1 + p] = (g.ndim == 2) ? ((P >> g.qx) | ((pl[iS] << g.shN) & g.rowL)) : 0;
            occ |= A[1 + p]; occx |= Bx[1 + p]; occy |= By[1 + p];
        }
        A[0] = g.valid & ~occ;
        Bx[0] = g.valid & ~occx;
        By[0] = g.valid & ~occy;
        const int ns = a.nplanes + 1;
        const int gy = g.row_offset + cy;
        int colour;
        if (a.C == 2) colour = g.ndim == 1 ? (cx & 1) : ((cx + gy) & 1);
        else colour = (cx & 1) + 2 * (gy & 1);
        for (int s = 0; s < ns; ++s) {
            const uint32_t c = __popcll(A[s]);
            acc[s] += c;
            acc[4 + colour * 4 + s] += c;
            for (int b = 0; b < ns; ++b) {
                acc[20 + s * 4 + b] += __popcll(A[s] & Bx[b]);
                if (g.ndim == 2) acc[20 + s * 4 + b] += __popcll(A[s] & By[b]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < kObsCounters; ++i) {
        const uint32_t v = __reduce_add_sync(0xffffffffu, acc[i]);
        if ((threadIdx.x & 31) == 0 && v) atomicAdd(&sh[i], (unsigned long long)v);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kObsCounters; i += blockDim.x)
        if (sh[i]) atomicAdd(&a.out[i], sh[i]);
}

cudaError_t launch_observables(const ObsArgs& a, cudaStream_t s) {
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const long long ncell = (long long)a.g.My_local * a.g.R * a.g.Mx;
    long long nb = (ncell + 255) / 256;
    if (nb > 4LL * nsm) nb = 4LL * nsm;
    if (nb < 1) nb = 1;
    observables_kernel<<<(unsigned)nb, 256, 0, s>>>(a);
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

}  // namespace kmc
