/*
 * kmc.h -- C ABI of the B200-native fractional-step kinetic Monte Carlo library
 * (libkmc_b200.so, built from paper_1105_4673_b200/csrc/).
 *
 * Method: Arampatzis, Katsoulakis, Plechac, Taufer, Xu, "Hierarchical
 * fractional-step approximations and parallel kinetic Monte Carlo algorithms"
 * (arXiv:1105.4673).  "P:n" = line n of the paper text; "R#" = the
 * readings listed in DESIGN.md §4; the arithmetic spec every result is
 * bit-exact to is DESIGN.md §3.
 *
 * The lattice generator L (eq.(generator)) is split over coarse
 * cells C_m (eq.(decomposition)) grouped into C colours
 * (eq.(sublatt); C = 4 for cross-cell-writing models, R6) and
 * advanced by a Lie (eq.(lie)), Strang (eq.(strang)) or
 * random sub-lattice (eq.(SLPCS)/eq.(SL)) product.  Inside one
 * window every cell of the active colour runs its own serial SSA
 * (eq.(exact); eq.(totalrate); eq.(skeleton)).
 *
 * Conventions (all entry points):
 *   - every call returns a kmc_status and never throws across the ABI; the
 *     last error text is kept per context (kmc_last_error) or, for a failed
 *     kmc_create, globally (kmc_create_error);
 *   - the context owns every device buffer it allocates; pointers passed in
 *     are borrowed for the duration of the call only;
 *   - host lattice buffers are uint8, site-major [replica][y][x] over the
 *     caller's LOCAL slab (rank-local rows in 2D, rank-local replicas in 1D);
 *     spin values: adsdes 0 vacant / 1 occupied; zgb 0 vacant / 1 CO / 2 O;
 *   - kmc_run / kmc_substep / kmc_*_device are stream-ordered and
 *     asynchronous on the context's stream; kmc_observables, kmc_set_config
 *     and kmc_get_config synchronise it.
 */
#ifndef KMC_B200_H
#define KMC_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kmc_ctx kmc_ctx;   /* opaque; owned by the library */

typedef enum {
    KMC_OK = 0,
    KMC_EINVAL = 1,       /* bad argument (NULL, unknown enum, spin value out of range, size mismatch) */
    KMC_EPARTITION = 2,   /* geometry violates R6/R7 (see kmc_create) */
    KMC_ENOMEM = 3,       /* device or host allocation failed */
    KMC_ECUDA = 4,        /* a CUDA runtime call or kernel failed (text in kmc_last_error) */
    KMC_ENCCL = 5,        /* an NCCL call failed or libnccl could not be loaded */
    KMC_ESTATE = 6,       /* call not valid in the context's current state */
    KMC_WTRUNCATED = 100  /* warning, kmc_run: T not a multiple of dt, last macro-step shortened (R20) */
} kmc_status;

typedef enum { KMC_LIE = 0, KMC_STRANG = 1, KMC_RANDOM = 2 } kmc_scheme;

/* Rate mechanisms.  Slot classes, canonical order:
 *  ADSDES       eq.(Arrhenius) P:963-968 (literal rates, R9):
 *               [adsorb c_a] [desorb c_d exp(-beta(K n + h)), n = 0..z]
 *  ADSDES_DIFF  + Kawasaki hops x->x+e_d, y vacant, c_hop exp(-beta K n(x)) (R12),
 *               d in (-x,+x,-y,+y), n = 0..z-1
 *  ZGB          Table COrates P:1132-1148 (R13): [CO adsorb k1] [O2 adsorb (1-k1)/z per
 *               vacant neighbour d] [CO+O react k2/z, CO anchor, d] [CO+O react k2/z, O anchor, d]
 *  ZGB_DIFF     + CO hops c_hop per vacant neighbour d
 *  ZGB_ODIFF    + O hops c_hop per vacant neighbour d: the fast O-adsorbate diffusion the paper's ZGB
 *               runs omit and its Strang scheme is meant to add (R33) -- the fast
 *               mechanism of kmc_run_multiscale by default
 *  z = 2 ndim.  */
typedef enum { KMC_ADSDES = 0, KMC_ADSDES_DIFF = 1, KMC_ZGB = 2, KMC_ZGB_DIFF = 3, KMC_ZGB_ODIFF = 4 } kmc_model_kind;

typedef struct {
    int32_t kind;                 /* kmc_model_kind */
    double ca, cd, beta, K, h;    /* Arrhenius ads/des (c1 = ca, c2 = cd) */
    double c_hop;                 /* hop prefactor (R12; ZGB_DIFF: CO hop rate; ZGB_ODIFF: O hop rate) */
    double k1, k2;                /* ZGB (R14) */
} kmc_model;

typedef struct {
    int32_t ndim;                 /* 1 or 2 */
    int64_t dims[2];              /* 1D: dims[0] = N sites.  2D: dims[0] = H rows (y), dims[1] = W cols (x) */
    int32_t cell[2];              /* 1D: cell[0] = Q.  2D: cell[0] = q_y, cell[1] = q_x;  q_x*q_y <= 64 */
    int32_t colours;              /* 0 = auto (2 for spin-flip or 1D, 4 otherwise), else 2 or 4 */
    int32_t replicas;             /* independent lattices batched (R21); global cell id = rep*M + m */
    uint64_t seed;                /* Philox key (R17) */
} kmc_geometry;

typedef struct {
    int32_t rank, world;          /* world = 1: single GPU.  world > 1: 2D slabs along y, 1D replicas split */
    int32_t device;               /* CUDA device ordinal */
    const uint8_t* nccl_unique_id;/* 128 bytes from kmc_nccl_unique_id() on rank 0, broadcast.  world = 1: NULL,
                                     or -- 2D only -- an id to run the lattice as a ONE-RANK PERIODIC RING
                                     through the multi-GPU data plane (NCCL loopback): ghost rows, the
                                     NCCL send/recv exchange with itself (and with fused_exchange = 1 the
                                     peer-write kernel variant and device flags on its own planes), so
                                     that transport executes on a single GPU; bit-identical to NULL */
    void* stream;                 /* cudaStream_t to launch on (e.g. torch's current stream); NULL = library-owned */
    const int64_t* row_bounds;    /* 2D, world > 1: world+1 cell-row bounds of the slabs (rank r owns cell rows
                                     [b_r, b_{r+1}), each an even number >= 2; e.g. from
                                     kmc_workload_partition), NULL = the even split.  Results do not depend
                                     on the split (global ids).  KMC_EPARTITION if invalid. */
    int32_t fused_exchange;       /* 2D, world > 1 (or the world = 1 loopback ring): 1 = fold the halo exchange into the window kernel (SURVEY
                                     §8(e)): the neighbours' planes are mapped with CUDA IPC (NVLink peer
                                     memory, one process per GPU on one node), the kernel writes the shared
                                     rows directly and windows are ordered by device-side flags instead of
                                     NCCL send/recv; bit-identical results.  0 = NCCL exchange (default).
                                     KMC_ECUDA if the IPC setup fails. */
} kmc_dist;

typedef struct {
    double time;                  /* physical time reached (sum of macro-step durations) */
    uint64_t windows;             /* global window (sub-step) counter, persists across kmc_run */
    uint64_t events;              /* executed SSA events since create (all ranks) */
    int64_t n_state[4];           /* sites per state (all ranks) */
    int64_t nn_pairs[4][4];       /* nearest-neighbour bonds {x,y} by unordered state pair, symmetric */
    int64_t n_state_by_colour[4][4]; /* [cell colour][state] */
    double coverage[4];           /* n_state / sites */
    double energy;                /* R24: -K nn_pairs[1][1] + h n_state[1] (paper H) */
} kmc_obs;

/* Create a context.  Validates the geometry (KMC_EPARTITION when: dims not divisible by the
 * cell, cell > 64 sites, odd number of cells per axis, cell extent < 2 for a cross-cell-writing
 * model (R7), 2 colours for a cross-cell-writing 2D model (R6), 2D rows per rank not a multiple of
 * 2 q_y, 1D replicas not divisible by world), builds the FP64 rate table and its u64 quantisation
 * (R18), allocates the bit-packed device lattice (all sites vacant, R22), and -- world > 1 --
 * initialises NCCL from the unique id.  On failure *out = NULL and kmc_create_error() explains. */
kmc_status kmc_create(const kmc_geometry* geom, const kmc_model* model, const kmc_dist* dist, kmc_ctx** out);
void kmc_destroy(kmc_ctx* ctx);
const char* kmc_last_error(const kmc_ctx* ctx);
const char* kmc_create_error(void);

/* Local slab sizes: bytes of the uint8 host/device lattice buffer this rank exchanges, and its
 * shape [replicas_local][rows_local][W] plus the global offsets of its first replica and row. */
kmc_status kmc_local_shape(const kmc_ctx* ctx, int64_t* replicas_local, int64_t* rows_local,
                           int64_t* width, int64_t* replica_offset, int64_t* row_offset);

/* Copy the local slab in (validating spin values < number of states, else KMC_EINVAL and the
 * lattice is unchanged) or out.  nbytes must equal replicas_local*rows_local*W.  Synchronous. */
/* Random initial configuration on the device (no upload; SURVEY §2.3 init kernel, reading R32):
 * every owned site (x, y) of replica r takes state s with probability probs[s] (nprobs = the
 * model's number of states; probs >= 0, partial sums <= 1, the last state takes the rest):
 * s = #{j < nprobs-1 : u >= T_j}, u = word 0 of Philox4x32-10((x, y, r, 2 << 28), key = seed),
 * T_j = floor(2^32 (probs[0] + .. + probs[j])), 2^32 once the sum reaches 1.  A site's state depends
 * on (seed, global coordinates) only: identical for any rank split.  Stream-ordered, asynchronous;
 * KMC_EINVAL on bad probabilities, KMC_ESTATE while a staged upload is pending. */
kmc_status kmc_init_random(kmc_ctx* ctx, const double* probs, int32_t nprobs, uint64_t seed);
kmc_status kmc_set_config(kmc_ctx* ctx, const uint8_t* host_local_slab, int64_t nbytes);
kmc_status kmc_get_config(kmc_ctx* ctx, uint8_t* host_local_slab, int64_t nbytes);
/* Same with a device buffer (e.g. a torch CUDA tensor), stream-ordered and asynchronous, so no
 * validation status: out-of-range spins are clamped to vacant and flagged; kmc_device_errors reports
 * whether the last kmc_set_config_device had any.  The lattice stays in the library's bit-packed
 * device planes (8x smaller than the uint8 buffer): the caller's buffer is read (set)
 * or written (get) during the call's stream work only and is never borrowed -- the uint8 site-major
 * layout of §8(b)'s borrowed kmc_dist.lattice cannot be the working layout of the bit-board kernels;
 * the borrowed buffer is the bit-packed working planes instead (kmc_attach_planes below). */
kmc_status kmc_set_config_device(kmc_ctx* ctx, const uint8_t* dev_local_slab, int64_t nbytes);
kmc_status kmc_get_config_device(kmc_ctx* ctx, uint8_t* dev_local_slab, int64_t nbytes);
/* Borrowed working lattice (§8(b)'s borrowed device buffer, in the kernels' own layout): after
 * kmc_attach_planes the windows, exchanges and observables run on the caller's device buffer
 * `dev_planes` (e.g. a torch int64 CUDA tensor's data_ptr, 8-byte aligned, on the context's device)
 * of nwords = planes x words_per_plane u64: plane p at dev_planes + p x words_per_plane, each plane
 * [storage row][replica][cell column] with storage rows = the owned cell rows plus, when the
 * context has ghost rows (2D, world > 1 or the loopback ring), one ghost row above and below
 * (owned row i at storage row i + ghost); a word's bit (ly*q_x + lx) is the site (cy*q_y + ly,
 * cx*q_x + lx) -- the kmc_set_config_packed layout plus the ghost rows.  The call copies the
 * current lattice in (stream-ordered) and frees the library's own planes; from then on the buffer
 * always holds the current lattice (configuration uploads copy into it instead of swapping
 * buffers) and it is never freed by the library: the caller keeps it alive until kmc_destroy.
 * kmc_planes_layout reports the sizes (before or after attaching).  KMC_EINVAL on a size mismatch
 * or a misaligned / NULL pointer; KMC_ESTATE with the fused exchange (its CUDA-IPC mappings are
 * made at create) or while a staged upload is pending. */
kmc_status kmc_planes_layout(const kmc_ctx* ctx, int32_t* planes, int64_t* words_per_plane, int64_t* storage_rows,
                             int32_t* ghost);
kmc_status kmc_attach_planes(kmc_ctx* ctx, uint64_t* dev_planes, int64_t nwords);
/* Bit-packed local slab (host buffers; the checkpoint format and the cheap upload path -- 1 bit per
 * site and plane instead of 1 byte per site): nwords = planes x rows_local/q_y x replicas_local x
 * W/q_x u64 words in the library's own layout [plane][cell row][replica][cell column] (DESIGN.md
 * §7): bit (ly*q_x + lx) of a word = site (cy*q_y + ly, cx*q_x + lx) of that replica.  Plane 0 =
 * occupied (ads/des models) or CO (ZGB); plane 1 = O (ZGB only).  set validates: bits beyond the
 * q_x*q_y sites of a cell, or a site both CO and O, give KMC_EINVAL and leave the lattice unchanged.
 * Synchronous. */
kmc_status kmc_set_config_packed(kmc_ctx* ctx, const uint64_t* host_words, int64_t nwords);
/* Pipelined upload of the next configuration (same packed layout and validation as
 * kmc_set_config_packed).  kmc_stage_config_packed enqueues the host->device copy into the
 * context's spare planes and the validation kernel on a separate copy stream and returns at once,
 * so the copy overlaps the windows already enqueued (the state they evolve is untouched);
 * kmc_commit_config then makes the staged configuration current, stream-ordered: windows enqueued
 * before the commit see the old lattice, windows after it the new one.  The host buffer must stay
 * valid and unchanged until kmc_commit_config returns (pinned memory gives a truly asynchronous
 * copy).  One stage may be pending: a second stage, kmc_set_config* while staged, or a commit
 * without a stage give KMC_ESTATE; a staged configuration that fails validation is discarded by
 * the commit with KMC_EINVAL (the current lattice is unchanged).  The commit waits (host) for the
 * staged copy and check only. */
kmc_status kmc_stage_config_packed(kmc_ctx* ctx, const uint64_t* host_words, int64_t nwords);
kmc_status kmc_commit_config(kmc_ctx* ctx);
kmc_status kmc_get_config_packed(kmc_ctx* ctx, uint64_t* host_words, int64_t nwords);
/* Asynchronous download of the current packed lattice (same layout as kmc_get_config_packed): the
 * device->host copy runs on the context's copy stream after everything enqueued so far and the call
 * returns at once; the host buffer (pinned for a truly asynchronous copy) holds the result after
 * kmc_download_wait (or kmc_destroy).  The device buffers being read are kept unchanged until the
 * copy ends: a later window, exchange or upload that would overwrite them waits for it on the
 * device, while windows that run on a configuration committed after the download
 * (kmc_stage_config_packed / kmc_commit_config swap other buffers in) overlap it.  A second download
 * first waits (host) for the previous one.  KMC_EINVAL on a size mismatch. */
kmc_status kmc_download_config_packed(kmc_ctx* ctx, uint64_t* host_words, int64_t nwords);
kmc_status kmc_download_wait(kmc_ctx* ctx);

/* Advance physical time by T with macro-steps of dt (R20: n = ceil(T/dt - 1e-9) macro-steps, the
 * last of duration T - (n-1) dt; KMC_WTRUNCATED if it differs from dt).  Lie: colours 0..C-1 for
 * dt each; Strang: palindrome with half steps for colour 0 (R2); random: C windows per macro-step,
 * colour xi_w drawn from Philox by global window id (R4).  Asynchronous. */
kmc_status kmc_run(kmc_ctx* ctx, double T, double dt, kmc_scheme scheme);

/* Temporal multiscale Strang (eq.(strang3)): per macro-step d,
 *   e^{d/2 L_slow} [ e^{(d/n_fast) L_fast} ]^{n_fast} e^{d/2 L_slow},
 * every factor itself split over the colours with the `inner` scheme (Lie, Strang or random, as in
 * kmc_run) -- the spatio-temporal hierarchy of P:750-753.  fast_classes: bit i = class i of the rate
 * table is fast (0 = the hop classes: ADSDES_DIFF's hops, ZGB_DIFF's CO or ZGB_ODIFF's O diffusion,
 * P:1211-1213).  Windows of one
 * mechanism run with the other mechanism's rates set to 0.  KMC_EINVAL when the fast set is empty or
 * covers every class; KMC_WTRUNCATED as kmc_run.  Asynchronous. */
kmc_status kmc_run_multiscale(kmc_ctx* ctx, double T, double dt, int32_t n_fast, kmc_scheme inner,
                              uint64_t fast_classes);

/* Nested two-level decomposition (eq.(sublatt2), eq.(opdecomp2), P:841-855;
 * DESIGN.md R28).  Outer blocks = `block` consecutive cell rows (2D; cells in 1D), coloured by block
 * parity (the paper's C_m^E / C_m^O); the cells inside are the paper's D_ml.  Per macro-step d the
 * outer Lie (0,d)(1,d) or Strang (0,d/2)(1,d)(0,d/2) factors; each outer factor of duration D is
 * n_inner cycles of the `inner` scheme (Lie, Strang, random) over the C cell colours, of duration
 * D/n_inner, restricted to the blocks of that outer colour.  With world > 1 the halo exchange runs
 * once per OUTER factor instead of once per window (blocks may not straddle ranks).  Errors:
 * KMC_EINVAL for outer = random, n_inner < 1, or an odd block / block < 2; KMC_EPARTITION when the
 * cells per axis are not a multiple of 2*block, or (world > 1) the local cell rows not a multiple
 * of block; KMC_WTRUNCATED as kmc_run.  Asynchronous. */
kmc_status kmc_run_nested(kmc_ctx* ctx, double T, double dt, int32_t n_inner, kmc_scheme outer, kmc_scheme inner,
                          int32_t block);

/* One window: every cell of colour `colour` runs its SSA for `duration` (eq.(exact)); the window
 * counter advances by one, physical time does not.  Asynchronous. */
kmc_status kmc_substep(kmc_ctx* ctx, int32_t colour, double duration);

/* Observables at the current state (a8).  per_cell_events (nullable, host) receives the
 * cumulative executed events of each LOCAL cell, uint32, in order [replica][cy][cx] (D5, eq.(wload)
 * the workload of a window is the difference of two snapshots).  Synchronous; world > 1
 * sums the counters over ranks (NCCL all-reduce). */
kmc_status kmc_observables(kmc_ctx* ctx, kmc_obs* out, uint32_t* per_cell_events);

/* Device-resident observables (a8 with no host round trip, e.g. once per macro-step inside a timed
 * or graph-captured loop): kmc_observables_device enqueues the counters of the current state into
 * dev_counters (KMC_OBS_WORDS uint64, caller-owned, in device memory of the context's device or in
 * pinned host memory, which a kernel then writes directly over the bus -- no copy-engine transfer
 * that would queue behind a pending kmc_download_config_packed; NCCL ranks all-reduce into device
 * memory first):
 * [0..3] sites per state, [4..19] sites per state by cell colour [colour*4 + state], [20..35]
 * ordered nearest-neighbour bonds (x, x+e), e in {+x, +y}, [a*4 + b], [36] events, [37] windows,
 * [38] time (IEEE double bits), [39] 0.  Stream-ordered, asynchronous; world > 1 sums words 0..36
 * over the NCCL ranks (collective).  kmc_obs_decode turns a host copy of those words into a kmc_obs
 * (what kmc_observables returns for the same state).  The vacant-state entries are completed from
 * the lattice identities (every site has one +e neighbour and is the +e neighbour of one site), so a
 * single virtual rank's words (kmc_vgroup_create) are contributions whose sum mod 2^64 over the
 * group is the count, not counts of that slab. */
#define KMC_OBS_WORDS 40
kmc_status kmc_observables_device(kmc_ctx* ctx, uint64_t* dev_counters);
/* Device-side error words (synchronises the context's stream): *bad_spins = 1 if the last
 * kmc_set_config_device held spin values >= the number of states (clamped to vacant);
 * *wait_timeouts = 1 if a fused-exchange flag wait gave up after 60 s (a neighbour rank never
 * arrived; the windows after it ran unordered and the state is void -- kmc_observables then returns
 * KMC_ECUDA).  Either pointer may be NULL. */
kmc_status kmc_device_errors(kmc_ctx* ctx, int32_t* bad_spins, int32_t* wait_timeouts);
kmc_status kmc_obs_decode(const kmc_ctx* ctx, const uint64_t* counters, kmc_obs* out);

/* Two-point correlation counts (the paper's 2-point correlation function
 * E[sigma_t(x) sigma_t(x+y)]): out_x[r] (r = 0..rmax) = number of sites x with
 * sigma(x) = state and sigma(x + r e_x) = state, summed over the whole lattice (periodic, all
 * replicas and ranks); out_y[r] the same along y (2D; zeros in 1D).  Divide by the number of sites
 * for E[1{sigma(x)=s} 1{sigma(x+r)=s}].  rmax must be < the lattice width (and height in 2D); with
 * world > 1, the y direction is limited to rmax <= q_y (one ghost cell row), else KMC_EINVAL.
 * Synchronous; the counts are exact integers. */
kmc_status kmc_correlation(kmc_ctx* ctx, int32_t rmax, int32_t state, int64_t* out_x, int64_t* out_y);

/* The coverage process C_t = |Lambda|^-1 sum_x 1{sigma_t(x) = state} of each replica (SURVEY §8(f)
 * f1; Figs. path1D, autocorr1D, pdf2d, dynamics2d: sample paths, autocorrelation function and
 * equilibrium distribution of the coverage; reading R30).
 *
 * kmc_record_coverage: (re)start recording.  Sample 0 is taken now; kmc_run, kmc_run_multiscale,
 *   kmc_run_nested and kmc_vgroup_run(_nested) append one sample at the end of every macro-step
 *   (including a shortened last one), on the device, stream-ordered, no host synchronisation.
 *   A sample is the per-LOCAL-replica number of sites in `state` (0 .. nstates-1) over the owned
 *   cells.  At most `capacity` samples are kept (later ones are dropped); capacity = 0 stops
 *   recording and frees the buffer.  KMC_EINVAL for a bad state or capacity < 0, KMC_ENOMEM.
 * kmc_coverage_series: copies min(max_samples, n) samples to `out` (host int64, [sample][local
 *   replica]) and sets *n_samples = n (out may be NULL to query n).  World > 1 over NCCL in 2D:
 *   the counts are summed over the rank slabs (complete per replica); 1D ranks own whole replicas.
 *   Virtual-rank contexts return their own slab's partial counts.  Synchronous.
 * kmc_coverage_stats: statistics of samples [first, n) over ALL replicas (all ranks), with
 *   c = count / sites-per-replica, M = replicas, n' = n - first:
 *     moments[0] = mean  c_bar = sum c / (M n');  moments[1] = gamma(0)
 *     gamma(l)   = sum_r sum_{i=first}^{n-1-l} (c_{i,r} - c_bar)(c_{i+l,r} - c_bar) / (M (n' - l))
 *     acf[l]     = gamma(l) / gamma(0) for l = 0..max_lag (all 0 when gamma(0) = 0)
 *     hist[b]    = #{(i, r) : floor(count_{i,r} * bins / (N + 1)) = b}, b < bins, N = sites per
 *                  replica (bins = N + 1: the exact distribution of N C_t)
 *   acf, moments, hist are host arrays (max_lag+1, 2, bins entries) and may each be NULL.
 *   KMC_EINVAL unless 0 <= first < n, 0 <= max_lag < n - first and (hist NULL or 1 <= bins <= N+1);
 *   KMC_ESTATE on a virtual-rank context.  Lag l is l macro-steps.  Synchronous; collective over
 *   NCCL ranks (every rank must call it). */
kmc_status kmc_record_coverage(kmc_ctx* ctx, int32_t state, int64_t capacity);
kmc_status kmc_coverage_series(kmc_ctx* ctx, int64_t* out, int64_t max_samples, int64_t* n_samples);
kmc_status kmc_coverage_stats(kmc_ctx* ctx, int64_t first, int32_t max_lag, double* acf, double* moments,
                              int32_t bins, int64_t* hist);

/* Checkpoint / resume: the whole state is (lattice, window counter, time, seed, config). */
kmc_status kmc_get_state(const kmc_ctx* ctx, uint64_t* windows, double* time);
kmc_status kmc_set_state(kmc_ctx* ctx, uint64_t windows, double time);

/* Inspection of the rate table (a1): n classes with type/dir/kappa, FP64 rate, u64 fixed point
 * and the scale exponent F (rate_u64 = llround(rate 2^F)).  Arrays hold >= 32 entries. */
kmc_status kmc_rate_table(const kmc_ctx* ctx, int32_t* n, int32_t* type, int32_t* dir, int32_t* kappa,
                          double* rate, uint64_t* rate_u64, int32_t* F);

/* Window-kernel choice (performance only; results are bit-identical):
 *   KMC_KERNEL_QUEUE: lane-per-cell kernel, per-warp cell queues, closure loaded from global memory;
 *   KMC_KERNEL_TILE:  2D spin-flip only -- a CTA stages a 32x64-cell tile + halo in shared memory and
 *                     runs its active cells from a CTA queue (best when a window holds few events);
 *   KMC_KERNEL_GROUPg (g = 2, 4, 8, 16, 32): spin flip only -- g lanes per cell: the g lanes draw g
 *                     consecutive events' random numbers in parallel and run the serial part of the
 *                     events in order (for windows with few active cells);
 *   KMC_KERNEL_AUTO:  spin flip: lane groups when a window's active cells fill less than a quarter
 *                     of the queue kernel's resident lanes (g = 2 or 4, measured best; env
 *                     KMC_GROUP=g forces g, 1 disables), else queue; other models: queue (env
 *                     KMC_TILE=0/1 overrides).
 * Nested windows (kmc_run_nested) and the fused cross-GPU exchange always use the queue kernel.
 * KMC_EINVAL for an unknown mode. */
typedef enum {
    KMC_KERNEL_AUTO = 0, KMC_KERNEL_QUEUE = 1, KMC_KERNEL_TILE = 2,
    KMC_KERNEL_GROUP2 = 3, KMC_KERNEL_GROUP4 = 4, KMC_KERNEL_GROUP8 = 5, KMC_KERNEL_GROUP16 = 6, KMC_KERNEL_GROUP32 = 7
} kmc_kernel_mode;
kmc_status kmc_set_kernel(kmc_ctx* ctx, int32_t mode);

/* Kernel timing (bench): when enabled, every sub-step kernel is bracketed by CUDA events on the
 * launching stream; kmc_timing returns the summed kernel milliseconds and launch count since the
 * last reset (synchronises). */
kmc_status kmc_enable_timing(kmc_ctx* ctx, int32_t enable);
kmc_status kmc_timing(kmc_ctx* ctx, double* kernel_ms, int64_t* launches, int32_t reset);

/* Host-side partition plan for rank `rank` of `world` (no device work): owned rows / replicas and
 * ring neighbours.  out[0] = replica_offset, out[1] = replicas_local, out[2] = row_offset,
 * out[3] = rows_local, out[4] = rank above (-y neighbour, -1 if none), out[5] = rank below. */
kmc_status kmc_partition_plan(const kmc_geometry* geom, int32_t kind, int32_t world, int32_t rank, int64_t out[6]);

/* Virtual ranks (single-GPU check of the multi-GPU path): create `world` contexts (ranks 0..world-1,
 * out[world]) holding the slabs of ONE 2D lattice on one device and stream, with exactly the slab
 * layout, ghost rows and exchange protocol of the NCCL path but the halo rows moved
 * by stream-ordered device copies.  kmc_vgroup_run advances all of them in lockstep (kmc_run and
 * kmc_substep on these contexts return KMC_ESTATE); kmc_vgroup_sync refreshes the ghost rows (call
 * it before kmc_observables, which then returns this rank's local counts, not the group sum).
 * Results are bit-identical to world = 1 (global ids).  Destroy each context with kmc_destroy. */
kmc_status kmc_vgroup_create(const kmc_geometry* geom, const kmc_model* model, int32_t world, int32_t device,
                             void* stream, kmc_ctx** out);
kmc_status kmc_vgroup_run(kmc_ctx** ctxs, int32_t world, double T, double dt, kmc_scheme scheme);
kmc_status kmc_vgroup_sync(kmc_ctx** ctxs, int32_t world);
/* Fused halo exchange on a virtual-rank group (the exchange folded into the window
 * kernel): enable != 0 makes every rank's window kernel mirror each write to a word of its first /
 * last owned cell row into the neighbour slab's ghost row, and each halo-delta XOR into a ghost row
 * into the neighbour's owned row (peer pointers to the other slabs' planes), so kmc_vgroup_run
 * performs no exchange between windows (one ghost refresh at the start of each call).  Results are
 * bit-identical to the exchange protocol and to world = 1.  Nested runs keep the exchange path.
 * While enabled, configuration uploads copy into the planes instead of swapping buffers. */
kmc_status kmc_vgroup_set_fused(kmc_ctx** ctxs, int32_t world, int32_t enable);
/* kmc_observables of the whole virtual-rank group (ghost rows refreshed first): the integer counters
 * and events summed over the ranks, coverage and energy (R24) decoded from the sums.  Synchronous. */
kmc_status kmc_vgroup_observables(kmc_ctx** ctxs, int32_t world, kmc_obs* out);
/* kmc_run_nested on a virtual-rank group (one exchange per outer factor). */
kmc_status kmc_vgroup_run_nested(kmc_ctx** ctxs, int32_t world, double T, double dt, int32_t n_inner,
                                 kmc_scheme outer, kmc_scheme inner, int32_t block);

/* kmc_vgroup_create with caller-chosen slabs (row_bounds as in kmc_dist; NULL = even split). */
kmc_status kmc_vgroup_create_bounds(const kmc_geometry* geom, const kmc_model* model, int32_t world, int32_t device,
                                    void* stream, const int64_t* row_bounds, kmc_ctx** out);

/* Workload re-balancing ("Mass Transport and Dynamic Workload Balancing",
 * P:885-940; R29).  The workload of eq.(wload) is the per-cell event count
 * since the last kmc_workload_mark (or since kmc_create).  It is summed over strips -- cell rows in
 * 2D (all columns and replicas), cells in 1D (all replicas) -- and the cdf of the strip
 * loads is mapped onto `parts` groups of equal mass: raw bound b_l = min{s+1 :
 * parts * cdf(s) >= l * S}, rounded to the nearest multiple of `granule` strips (ties up) and
 * clamped so that every group keeps >= granule strips; no events gives the even split.
 * bounds (host, parts+1 entries) receives b_0 = 0 < ... < b_parts = strips; in 2D with granule 2
 * they are valid kmc_dist.row_bounds for `parts` ranks.  strip_load (host, nullable, one u64 per
 * strip) receives the loads; imbalance (host, nullable, 2 doubles) = max group load x parts / S for
 * the cdf bounds and for the even split.  world > 1: the strip loads are summed over ranks (NCCL),
 * every rank gets the same bounds.  KMC_EINVAL: parts outside [1, 4096], strips not a multiple of
 * granule or fewer than parts*granule.  Requires parts * S < 2^64.  Synchronous. */
kmc_status kmc_workload_mark(kmc_ctx* ctx);
kmc_status kmc_workload_partition(kmc_ctx* ctx, int32_t parts, int32_t granule, int64_t* bounds, uint64_t* strip_load,
                                  double* imbalance);
/* The same over a virtual-rank group (strip loads of all ranks). */
kmc_status kmc_vgroup_workload_partition(kmc_ctx** ctxs, int32_t world, int32_t parts, int32_t granule, int64_t* bounds,
                                         uint64_t* strip_load, double* imbalance);

/* NCCL unique id for world > 1 (rank 0 calls it and broadcasts the 128 bytes). */
kmc_status kmc_nccl_unique_id(uint8_t out[128]);

/* Library version string. */
const char* kmc_version(void);

/* ABI check (host only, no device): out[0..3] = sizeof(kmc_geometry), sizeof(kmc_model),
 * sizeof(kmc_dist), sizeof(kmc_obs), so bindings can verify their struct layouts. */
void kmc_abi_sizes(int64_t out[4]);

#ifdef __cplusplus
}
#endif
#endif /* KMC_B200_H */
