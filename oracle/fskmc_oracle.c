/*
 * fskmc_oracle.c -- CPU ORACLE for the fractional-step KMC hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code with paper_1105_4673_b200/ (the CUDA product path) and
 * neither side includes or links the other.
 *
 * Paper: Arampatzis, Katsoulakis, Plechac, Taufer, Xu, "Hierarchical
 * fractional-step approximations and parallel kinetic Monte Carlo
 * algorithms" (arXiv:1105.4673).  Citations "P:n" are lines of
 * /root/reference/PAPER.md; "R#" are the readings listed in DESIGN.md §4.
 *
 * Contents
 *   O2  orc_window()     one fractional-step window e^{D L^c} (eq.(exact),
 *                        P:402-417): every cell of colour c runs its own
 *                        serial SSA (eq.(totalrate), eq.(skeleton)
 *                        P:106-108) for time D.  Written as a plain linear
 *                        scan over the canonical slot list.
 *   O1  orc_ssa()        exact serial SSA on the whole lattice (the CTMC of
 *                        eq.(generator)), Fenwick-tree selection,
 *                        an RNG stream disjoint from O2's.
 *   L0  orc_philox4x32_10, orc_log   the arithmetic spec.
 *   a1  orc_classes / orc_quantise   the rate table (eq.(Arrhenius)
 *                        P:963-968, Table COrates, R12-R14, R18).
 *
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no FMA contraction: the
 * clock arithmetic must be the IEEE operation sequence of DESIGN.md §3).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* L0: Philox4x32-10 (Salmon et al., SC'11; Random123 constants).      */
/* ------------------------------------------------------------------ */
void orc_philox4x32_10(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4])
{
    uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
    uint32_t k0 = key_in[0], k1 = key_in[1];
    for (int round = 0; round < 10; ++round) {
        uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
        uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t n0 = hi1 ^ c1 ^ k0;
        uint32_t n1 = lo1;
        uint32_t n2 = hi0 ^ c3 ^ k1;
        uint32_t n3 = lo0;
        c0 = n0; c1 = n1; c2 = n2; c3 = n3;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

/* ------------------------------------------------------------------ */
/* L0: natural log, table-driven, every step one       */
/* correctly rounded IEEE operation (C99 fma() for the fused steps).    */
/*   x = 2^e m, m in [sqrt(2)/2, sqrt(2));  j = round(128 m) - 91;      */
/*   c_j = 128/(j+91), L_j = -log(c_j) (host libm);                      */
/*   r = fma(m, c_j, -1);  log x = e ln2 + L_j + log1p(r),               */
/*   log1p(r) = r + r^2 q(r), q the Taylor polynomial to r^7 (Horner).   */
/* Domain: normal x in (0, 1] (the clock only needs [2^-53, 1]).         */
/* ------------------------------------------------------------------ */
static const double ln2_hi = 0x1.62e42feep-1;          /* 3fe62e42 fee00000 */
static const double ln2_lo = 0x1.a39ef35793c76p-33;    /* 3dea39ef 35793c76 */
#define LOG_TAB_N 91
static double log_ctab[LOG_TAB_N], log_ltab[LOG_TAB_N];
static int log_tab_ready = 0;

static inline uint64_t dbits(double x) { uint64_t u; memcpy(&u, &x, 8); return u; }
static inline double bitsd(uint64_t u) { double x; memcpy(&x, &u, 8); return x; }

static void log_tables(void)
{
    for (int j = 0; j < LOG_TAB_N; ++j) {
        log_ctab[j] = 128.0 / (double)(j + 91);
        log_ltab[j] = -log(log_ctab[j]);
    }
    log_tab_ready = 1;
}

double orc_log(double x)
{
    if (!log_tab_ready) log_tables();
    if (x == 0.0) return -INFINITY;
    uint64_t u = dbits(x);
    int e0 = (int)((u >> 52) & 0x7ff) - 1023;
    if (e0 == -1023 || e0 == 1024 || (u >> 63)) return NAN;      /* outside the specified domain */
    uint64_t mant = u & 0xFFFFFFFFFFFFFull;
    int e, idx;
    double m;
    if (mant >= 0x6A09E667F3BCDull) {                             /* 1.mant >= sqrt(2): halve */
        e = e0 + 1;
        idx = 64 + (int)((mant + (1ull << 45)) >> 46);
        m = bitsd(0x3FE0000000000000ull | mant);
    } else {
        e = e0;
        idx = 128 + (int)((mant + (1ull << 44)) >> 45);
        m = bitsd(0x3FF0000000000000ull | mant);
    }
    const int j = idx - 91;
    const double r = fma(m, log_ctab[j], -1.0);
    double q = fma(r, 0x1.2492492492492p-3, -0x1.5555555555555p-3);    /* 1/7, -1/6 */
    q = fma(r, q, 0x1.999999999999ap-3);                                 /* 1/5 */
    q = fma(r, q, -0.25);
    q = fma(r, q, 0x1.5555555555555p-2);                                 /* 1/3 */
    q = fma(r, q, -0.5);
    const double p = fma(r * r, q, r);
    const double dk = (double)e;
    double s = log_ltab[j] + p;
    s = fma(dk, ln2_lo, s);
    return fma(dk, ln2_hi, s);
}

/* ------------------------------------------------------------------ */
/* Models, slot types and the canonical class list.   */
/* ------------------------------------------------------------------ */
enum { M_ADSDES = 0, M_ADSDES_DIFF = 1, M_ZGB = 2, M_ZGB_DIFF = 3, M_ZGB_ODIFF = 4 };
enum { T_ADS = 0, T_DES = 1, T_HOP = 2, T_COADS = 3, T_O2ADS = 4, T_RCO = 5, T_RO = 6, T_COHOP = 7, T_OHOP = 8 };
#define MAXCLASS 32

/* params[] = {ca, cd, beta, K, h, c_hop, k1, k2} */
int orc_classes(int kind, int ndim, const double* params,
                int* ctype, int* cdir, int* ckappa, double* crate)
{
    const double ca = params[0], cd = params[1], beta = params[2], K = params[3];
    const double h = params[4], chop = params[5], k1 = params[6], k2 = params[7];
    const int z = 2 * ndim;             /* coordination number */
    int n = 0;
    if (kind == M_ADSDES || kind == M_ADSDES_DIFF) {
        /* eq.(Arrhenius): c = c1 (1-s) + c2 s exp(-beta U), U = K n + h  (R9: literal) */
        ctype[n] = T_ADS; cdir[n] = -1; ckappa[n] = 0; crate[n] = ca; ++n;
        for (int m = 0; m <= z; ++m) {
            double t = K * (double)m;
            t = t + h;
            t = beta * t;
            t = -t;
            ctype[n] = T_DES; cdir[n] = -1; ckappa[n] = m; crate[n] = cd * exp(t); ++n;
        }
        if (kind == M_ADSDES_DIFF) {
            /* R12: hop x->y (y vacant) at c_hop exp(-beta K n(x)); R31: classes n-major
             * (n(x) = 0..z-1 outer, direction d inner) */
            for (int m = 0; m <= z - 1; ++m)
                for (int d = 0; d < z; ++d) {
                    double t = K * (double)m;
                    t = beta * t;
                    t = -t;
                    ctype[n] = T_HOP; cdir[n] = d; ckappa[n] = m; crate[n] = chop * exp(t); ++n;
                }
        }
        return n;
    }
    if (kind == M_ZGB || kind == M_ZGB_DIFF || kind == M_ZGB_ODIFF) {
        /* Table COrates, storage 0 vacant, 1 CO, 2 O (R13); one slot per direction (R13) */
        ctype[n] = T_COADS; cdir[n] = -1; ckappa[n] = 0; crate[n] = k1; ++n;
        for (int d = 0; d < z; ++d) { ctype[n] = T_O2ADS; cdir[n] = d; ckappa[n] = 0; crate[n] = (1.0 - k1) / (double)z; ++n; }
        for (int d = 0; d < z; ++d) { ctype[n] = T_RCO;   cdir[n] = d; ckappa[n] = 0; crate[n] = k2 / (double)z; ++n; }
        for (int d = 0; d < z; ++d) { ctype[n] = T_RO;    cdir[n] = d; ckappa[n] = 0; crate[n] = k2 / (double)z; ++n; }
        if (kind == M_ZGB_DIFF)
            for (int d = 0; d < z; ++d) { ctype[n] = T_COHOP; cdir[n] = d; ckappa[n] = 0; crate[n] = chop; ++n; }
        /* the fast O-adsorbate diffusion the paper leaves out of ZGB (after \cite{evans09}):
         * O(x), vacant y = x + e_d -> vacant, O at c_hop per vacant neighbour direction (R33) */
        if (kind == M_ZGB_ODIFF)
            for (int d = 0; d < z; ++d) { ctype[n] = T_OHOP; cdir[n] = d; ckappa[n] = 0; crate[n] = chop; ++n; }
        return n;
    }
    return -1;
}

/* slot types per site (upper bound on simultaneously eligible slots at one anchor) */
int orc_types_per_site(int kind, int ndim)
{
    int z = 2 * ndim;
    switch (kind) {
    case M_ADSDES: return 2;
    case M_ADSDES_DIFF: return 2 + z;
    case M_ZGB: return 1 + 3 * z;
    case M_ZGB_DIFF: return 1 + 4 * z;
    case M_ZGB_ODIFF: return 1 + 4 * z;
    }
    return -1;
}

/* R18: F = 62 - ceil(log2(S_max * r_max)); rate_u64 = llround(rate * 2^F). Returns F (or -1). */
int orc_quantise(const double* crate, int n, int sites_per_cell, int types_per_site, uint64_t* out)
{
    double rmax = 0.0;
    for (int c = 0; c < n; ++c) {
        if (!(crate[c] >= 0.0) || isinf(crate[c])) return -1;
        if (crate[c] > rmax) rmax = crate[c];
    }
    int F;
    if (rmax == 0.0) F = 0;
    else {
        double bound = rmax * (double)((int64_t)sites_per_cell * types_per_site);
        int e;
        double m = frexp(bound, &e);         /* bound = m 2^e, m in [0.5, 1) */
        int cl = (m == 0.5) ? e - 1 : e;     /* ceil(log2(bound)) */
        F = 62 - cl;
        if (F < 0) return -1;
    }
    for (int c = 0; c < n; ++c) out[c] = (uint64_t)llround(ldexp(crate[c], F));
    return F;
}

/* ------------------------------------------------------------------ */
/* Lattice helpers: uint8 site-major [R][H][W], periodic.              */
/* ------------------------------------------------------------------ */
typedef struct {
    uint8_t* lat; int64_t H, W; int ndim;
} latview;

static inline uint8_t get_site(const latview* L, int64_t rep, int64_t y, int64_t x)
{
    y = (y % L->H + L->H) % L->H;
    x = (x % L->W + L->W) % L->W;
    return L->lat[(rep * L->H + y) * L->W + x];
}
static inline void set_site(latview* L, int64_t rep, int64_t y, int64_t x, uint8_t v)
{
    y = (y % L->H + L->H) % L->H;
    x = (x % L->W + L->W) % L->W;
    L->lat[(rep * L->H + y) * L->W + x] = v;
}
/* direction d: 0 -x, 1 +x, 2 -y, 3 +y */
static const int DX[4] = {-1, +1, 0, 0};
static const int DY[4] = {0, 0, -1, +1};

/* number of nearest neighbours of (y,x) in state v */
static int count_nbrs(const latview* L, int64_t rep, int64_t y, int64_t x, uint8_t v)
{
    int z = 2 * L->ndim, n = 0;
    for (int d = 0; d < z; ++d)
        n += get_site(L, rep, y + DY[d], x + DX[d]) == v;
    return n;
}

/* Is slot (type, dir) eligible at anchor (y,x), and with which kappa? */
static int slot_kappa(const latview* L, int64_t rep, int64_t y, int64_t x, int type, int dir, int* kappa)
{
    uint8_t s = get_site(L, rep, y, x);
    uint8_t p = 0;
    if (dir >= 0) p = get_site(L, rep, y + DY[dir], x + DX[dir]);
    *kappa = 0;
    switch (type) {
    case T_ADS: return s == 0;
    case T_DES: if (s != 1) return 0; *kappa = count_nbrs(L, rep, y, x, 1); return 1;
    case T_HOP: if (!(s == 1 && p == 0)) return 0; *kappa = count_nbrs(L, rep, y, x, 1); return 1;
    case T_COADS: return s == 0;
    case T_O2ADS: return s == 0 && p == 0;
    case T_RCO: return s == 1 && p == 2;
    case T_RO: return s == 2 && p == 1;
    case T_COHOP: return s == 1 && p == 0;
    case T_OHOP: return s == 2 && p == 0;
    }
    return 0;
}

static void apply_slot(latview* L, int64_t rep, int64_t y, int64_t x, int type, int dir)
{
    int64_t py = 0, px = 0;
    if (dir >= 0) { py = y + DY[dir]; px = x + DX[dir]; }
    switch (type) {
    case T_ADS:   set_site(L, rep, y, x, 1); break;
    case T_DES:   set_site(L, rep, y, x, 0); break;
    case T_HOP:   set_site(L, rep, y, x, 0); set_site(L, rep, py, px, 1); break;
    case T_COADS: set_site(L, rep, y, x, 1); break;
    case T_O2ADS: set_site(L, rep, y, x, 2); set_site(L, rep, py, px, 2); break;
    case T_RCO:   set_site(L, rep, y, x, 0); set_site(L, rep, py, px, 0); break;
    case T_RO:    set_site(L, rep, y, x, 0); set_site(L, rep, py, px, 0); break;
    case T_COHOP: set_site(L, rep, y, x, 0); set_site(L, rep, py, px, 1); break;
    case T_OHOP:  set_site(L, rep, y, x, 0); set_site(L, rep, py, px, 2); break;
    }
}

/* colour of cell (cy,cx): R6 */
int orc_cell_colour(int ndim, int C, int64_t cy, int64_t cx)
{
    if (C == 2) return ndim == 1 ? (int)(cx & 1) : (int)((cx + cy) & 1);
    return (int)(cx & 1) + 2 * (int)(cy & 1);
}

/* ------------------------------------------------------------------ */
/* O2: one window for ONE cell (r, cy, cx): the serial SSA of the cell for time D.  */
/* Returns the number of executed events.                                          */
/* ------------------------------------------------------------------ */
static uint32_t cell_window(latview* L, int64_t rep, int64_t cy, int64_t cx, int qx, int qy,
                            uint64_t gid, double D, uint64_t window, const uint32_t key[2],
                            int nclass, const int* ctype, const int* cdir, const int* ckappa,
                            const uint64_t* crate_u64, double inv_scale)
{
    const int nsite = qx * qy;
    /* member[c][s] = 1 if slot class c is eligible at local site s */
    uint8_t member[MAXCLASS][64];
    double t = 0.0;
    uint32_t k = 0;
    for (;;) {
        /* eq.(totalrate) restricted to the cell: enumerate slots in canonical order */
        uint64_t cnt[MAXCLASS];
        uint64_t lam = 0;
        for (int c = 0; c < nclass; ++c) {
            cnt[c] = 0;
            for (int s = 0; s < nsite; ++s) {
                int64_t y = cy * qy + s / qx, x = cx * qx + s % qx;
                int kap;
                int el = slot_kappa(L, rep, y, x, ctype[c], cdir[c], &kap) && kap == ckappa[c];
                member[c][s] = (uint8_t)el;
                cnt[c] += (uint64_t)el;
            }
            lam += cnt[c] * crate_u64[c];
        }
        if (lam == 0) break;                               /* quiescent cell */
        uint32_t ctr[4] = {k, (uint32_t)gid, (uint32_t)window,
                           (uint32_t)((window >> 32) & 0x0FFFFFFFu) | (0u << 28)};
        uint32_t xr[4];
        orc_philox4x32_10(ctr, key, xr);
        /* exponential clock, eq.(totalrate): tau = -ln U / lambda */
        uint64_t j53 = ((uint64_t)xr[0] << 21) | (uint64_t)(xr[1] >> 11);
        double U = (double)(j53 + 1) * 0x1p-53;
        double E = -orc_log(U);
        double lamd = (double)lam * inv_scale;
        double tau = E / lamd;
        if (t + tau >= D) break;                           /* R5: pending event discarded */
        t = t + tau;
        /* eq.(skeleton): class with prob cnt*rate/lambda, then a uniform member site */
        uint64_t r = (uint64_t)(((unsigned __int128)xr[2] * (unsigned __int128)lam) >> 32);
        uint64_t cum = 0;
        int csel = -1;
        for (int c = 0; c < nclass; ++c) {
            cum += cnt[c] * crate_u64[c];
            if (cum > r) { csel = c; break; }
        }
        uint64_t kk = ((uint64_t)xr[3] * cnt[csel]) >> 32;
        int ssel = -1;
        uint64_t seen = 0;
        for (int s = 0; s < nsite; ++s) {
            if (member[csel][s]) {
                if (seen == kk) { ssel = s; break; }
                ++seen;
            }
        }
        int64_t y = cy * qy + ssel / qx, x = cx * qx + ssel % qx;
        apply_slot(L, rep, y, x, ctype[csel], cdir[csel]);
        ++k;
    }
    return k;
}

/* O2: one window of colour `colour` and duration D on all replicas (eq.(exact): the cells of
 * one colour are independent, so processing them in any order in place is exact).
 * Returns the number of executed events; W_events[gid] += events. */
int64_t orc_window(uint8_t* lat, int R, int64_t H, int64_t W, int ndim, int qx, int qy,
                   int C, int colour, double D, uint64_t window, uint64_t seed,
                   int nclass, const int* ctype, const int* cdir, const int* ckappa,
                   const uint64_t* crate_u64, int F, uint32_t* W_events)
{
    latview L = {lat, H, W, ndim};
    const int64_t Mx = W / qx, My = H / qy;
    const double inv_scale = ldexp(1.0, -F);          /* 2^-F */
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int64_t total = 0;
    /* The cells of one colour are independent within a window (eq.(exact); same-colour
     * closures are disjoint, R6), so the timing build (tools/oracle_timing.py, -fopenmp) runs them
     * on all host cores with identical results; the test build is single-threaded. */
#ifdef _OPENMP
#pragma omp parallel for reduction(+ : total) schedule(dynamic, 64)
#endif
    for (int64_t t = 0; t < (int64_t)R * My * Mx; ++t) {
        const int64_t rep = t / (My * Mx), cy = (t / Mx) % My, cx = t % Mx;
        if (orc_cell_colour(ndim, C, cy, cx) != colour) continue;
        const uint64_t gid = (uint64_t)rep * (uint64_t)(Mx * My) + (uint64_t)(cy * Mx + cx);
        uint32_t k = cell_window(&L, rep, cy, cx, qx, qy, gid, D, window, key,
                                 nclass, ctype, cdir, ckappa, crate_u64, inv_scale);
        if (W_events) W_events[gid] += k;
        total += k;
    }
    return total;
}

/* O2 on a LIST of cells (cells[3*i] = replica, cy, cx), all of one colour: used to check sampled
 * cells of a full-size GPU window against the pre-window lattice.  events_out[i] = events. */
int64_t orc_window_cells(uint8_t* lat, int R, int64_t H, int64_t W, int ndim, int qx, int qy,
                         const int64_t* cells, int64_t ncells, double D, uint64_t window, uint64_t seed,
                         int nclass, const int* ctype, const int* cdir, const int* ckappa,
                         const uint64_t* crate_u64, int F, uint32_t* events_out)
{
    latview L = {lat, H, W, ndim};
    const int64_t Mx = W / qx, My = H / qy;
    const double inv_scale = ldexp(1.0, -F);
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    int64_t total = 0;
    (void)R;
    for (int64_t i = 0; i < ncells; ++i) {
        const int64_t rep = cells[3 * i], cy = cells[3 * i + 1], cx = cells[3 * i + 2];
        const uint64_t gid = (uint64_t)rep * (uint64_t)(Mx * My) + (uint64_t)(cy * Mx + cx);
        uint32_t k = cell_window(&L, rep, cy, cx, qx, qy, gid, D, window, key,
                                 nclass, ctype, cdir, ckappa, crate_u64, inv_scale);
        if (events_out) events_out[i] = k;
        total += k;
    }
    return total;
}

/* ------------------------------------------------------------------ */
/* O1: exact serial SSA on one replica (whole lattice), eq.(generator). */
/* Slot index = site * ntype + type_slot, where the per-site slot types  */
/* are the distinct (type,dir) pairs of the class list.  Fenwick tree of */
/* u64 fixed-point rates (exact sums).  Records the lattice at the given */
/* observation times (state just before the first event after T_obs).    */
/* RNG: Philox keyed by seed, counter (n_lo, n_hi, stream, 3<<28).       */
/* ------------------------------------------------------------------ */
typedef struct { int type, dir; } slotdef;

static void fen_add(uint64_t* tree, int64_t n, int64_t i, uint64_t delta_add, int neg)
{
    for (++i; i <= n; i += i & (-i)) {
        if (neg) tree[i] -= delta_add; else tree[i] += delta_add;
    }
}

int64_t orc_ssa(uint8_t* lat, int64_t H, int64_t W, int ndim,
                int nclass, const int* ctype, const int* cdir, const int* ckappa,
                const uint64_t* crate_u64, int F, uint64_t seed, uint32_t stream,
                const double* T_obs, int n_obs, uint8_t* out_snapshots)
{
    latview L = {lat, H, W, ndim};
    const int64_t N = H * W;
    slotdef defs[MAXCLASS];
    int ntype = 0;
    for (int c = 0; c < nclass; ++c) {
        int found = 0;
        for (int j = 0; j < ntype; ++j) if (defs[j].type == ctype[c] && defs[j].dir == cdir[c]) found = 1;
        if (!found) { defs[ntype].type = ctype[c]; defs[ntype].dir = cdir[c]; ++ntype; }
    }
    const int64_t nslot = N * ntype;
    uint64_t* rate = (uint64_t*)calloc((size_t)nslot, sizeof(uint64_t));
    uint64_t* tree = (uint64_t*)calloc((size_t)nslot + 1, sizeof(uint64_t));
    if (!rate || !tree) { free(rate); free(tree); return -1; }
    int64_t top = 1;
    while (top * 2 <= nslot) top *= 2;

    /* rate of a slot (site, j) */
#define SLOT_RATE(site, j, outv) do { \
        int64_t yy_ = (site) / W, xx_ = (site) % W; int kap_; \
        uint64_t rr_ = 0; \
        if (slot_kappa(&L, 0, yy_, xx_, defs[j].type, defs[j].dir, &kap_)) { \
            for (int c_ = 0; c_ < nclass; ++c_) \
                if (ctype[c_] == defs[j].type && cdir[c_] == defs[j].dir && ckappa[c_] == kap_) { rr_ = crate_u64[c_]; break; } \
        } \
        (outv) = rr_; } while (0)

    for (int64_t s = 0; s < N; ++s)
        for (int j = 0; j < ntype; ++j) {
            uint64_t v; SLOT_RATE(s, j, v);
            rate[s * ntype + j] = v;
            fen_add(tree, nslot, s * ntype + j, v, 0);
        }
    uint64_t lam = 0;
    for (int64_t i = 0; i < nslot; ++i) lam += rate[i];

    const double inv_scale = ldexp(1.0, -F);
    const uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
    double t = 0.0;
    uint64_t nev = 0;
    int obs = 0;
    while (obs < n_obs) {
        double tau;
        uint32_t xr[4];
        if (lam == 0) tau = INFINITY;
        else {
            uint32_t ctr[4] = {(uint32_t)nev, (uint32_t)(nev >> 32), stream, 3u << 28};
            orc_philox4x32_10(ctr, key, xr);
            uint64_t j53 = ((uint64_t)xr[0] << 21) | (uint64_t)(xr[1] >> 11);
            double U = (double)(j53 + 1) * 0x1p-53;
            tau = -orc_log(U) / ((double)lam * inv_scale);
        }
        while (obs < n_obs && t + tau > T_obs[obs]) {
            memcpy(out_snapshots + (size_t)obs * (size_t)N, lat, (size_t)N);
            ++obs;
        }
        if (obs >= n_obs) break;
        t += tau;
        uint64_t v = ((uint64_t)xr[2] << 32) | xr[3];
        uint64_t r = (uint64_t)(((unsigned __int128)v * (unsigned __int128)lam) >> 64);
        /* Fenwick descent: smallest i with prefix(i) > r */
        int64_t pos = 0;
        uint64_t rem = r;
        for (int64_t step = top; step > 0; step >>= 1) {
            if (pos + step <= nslot && tree[pos + step] <= rem) { pos += step; rem -= tree[pos]; }
        }
        int64_t slot = pos;                     /* 0-based */
        int64_t site = slot / ntype;
        int j = (int)(slot % ntype);
        int64_t y = site / W, x = site % W;
        apply_slot(&L, 0, y, x, defs[j].type, defs[j].dir);
        ++nev;
        /* refresh all slots anchored within distance 2 of the anchor (covers partner's ball) */
        for (int64_t dy = -2; dy <= 2; ++dy)
            for (int64_t dx = -2; dx <= 2; ++dx) {
                if (ndim == 1 && dy != 0) continue;
                if (llabs(dy) + llabs(dx) > 2) continue;
                int64_t yy = ((y + dy) % H + H) % H, xx = ((x + dx) % W + W) % W;
                int64_t s2 = yy * W + xx;
                for (int j2 = 0; j2 < ntype; ++j2) {
                    uint64_t nv; SLOT_RATE(s2, j2, nv);
                    uint64_t ov = rate[s2 * ntype + j2];
                    if (nv != ov) {
                        if (nv > ov) { fen_add(tree, nslot, s2 * ntype + j2, nv - ov, 0); lam += nv - ov; }
                        else { fen_add(tree, nslot, s2 * ntype + j2, ov - nv, 1); lam -= ov - nv; }
                        rate[s2 * ntype + j2] = nv;
                    }
                }
            }
    }
#undef SLOT_RATE
    free(rate); free(tree);
    return (int64_t)nev;
}
