"""B200-native fractional-step kinetic Monte Carlo (arXiv:1105.4673) -- Python binding.

A thin ctypes layer over the C ABI of ``libkmc_b200.so`` (include/kmc.h): argument
marshalling only.  Every step of the hot path (rate table, schedule, per-cell SSA
windows, halo exchange, observables) runs in the library and its sm_100a kernels;
there is no CPU fallback -- if the library is missing this module raises.
PyTorch is used only for device memory, streams and process groups.
"""
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libkmc_b200.so")
# A/B performance comparisons may point at another in-tree build of the same library
LIB_PATH = os.environ.get("KMC_B200_LIB", LIB_PATH)

KMC_OK, KMC_EINVAL, KMC_EPARTITION, KMC_ENOMEM, KMC_ECUDA, KMC_ENCCL, KMC_ESTATE = 0, 1, 2, 3, 4, 5, 6
KMC_WTRUNCATED = 100
SCHEMES = {"lie": 0, "strang": 1, "random": 2}
KINDS = {"adsdes": 0, "adsdes_diff": 1, "zgb": 2, "zgb_diff": 3, "zgb_odiff": 4}
NSTATES = {0: 2, 1: 2, 2: 3, 3: 3, 4: 3}

# Every symbol include/kmc.h declares (checked by tests/test_abi.py).
EXPORTS = [
    "kmc_create", "kmc_destroy", "kmc_last_error", "kmc_create_error", "kmc_local_shape",
    "kmc_set_config", "kmc_get_config", "kmc_set_config_device", "kmc_get_config_device",
    "kmc_planes_layout", "kmc_attach_planes",
    "kmc_run", "kmc_substep", "kmc_observables", "kmc_get_state", "kmc_set_state",
    "kmc_rate_table", "kmc_enable_timing", "kmc_timing", "kmc_partition_plan",
    "kmc_nccl_unique_id", "kmc_version", "kmc_vgroup_create", "kmc_vgroup_run", "kmc_vgroup_sync",
    "kmc_set_kernel", "kmc_correlation", "kmc_run_multiscale", "kmc_run_nested",
    "kmc_vgroup_run_nested", "kmc_set_config_packed", "kmc_get_config_packed",
    "kmc_vgroup_create_bounds", "kmc_workload_mark", "kmc_workload_partition", "kmc_vgroup_workload_partition",
    "kmc_vgroup_set_fused", "kmc_abi_sizes", "kmc_record_coverage", "kmc_coverage_series", "kmc_coverage_stats",
    "kmc_stage_config_packed", "kmc_commit_config", "kmc_observables_device", "kmc_obs_decode",
    "kmc_init_random", "kmc_device_errors", "kmc_vgroup_observables", "kmc_download_config_packed",
    "kmc_download_wait",
]
OBS_WORDS = 40
KERNELS = {"auto": 0, "queue": 1, "tile": 2, "group2": 3, "group4": 4, "group8": 5, "group16": 6, "group32": 7}


class KmcModel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("ca", ctypes.c_double), ("cd", ctypes.c_double),
                ("beta", ctypes.c_double), ("K", ctypes.c_double), ("h", ctypes.c_double),
                ("c_hop", ctypes.c_double), ("k1", ctypes.c_double), ("k2", ctypes.c_double)]


class KmcGeometry(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int32), ("dims", ctypes.c_int64 * 2), ("cell", ctypes.c_int32 * 2),
                ("colours", ctypes.c_int32), ("replicas", ctypes.c_int32), ("seed", ctypes.c_uint64)]


class KmcDist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("nccl_unique_id", ctypes.c_void_p), ("stream", ctypes.c_void_p), ("row_bounds", ctypes.c_void_p),
                ("fused_exchange", ctypes.c_int32)]


class KmcObs(ctypes.Structure):
    _fields_ = [("time", ctypes.c_double), ("windows", ctypes.c_uint64), ("events", ctypes.c_uint64),
                ("n_state", ctypes.c_int64 * 4), ("nn_pairs", (ctypes.c_int64 * 4) * 4),
                ("n_state_by_colour", (ctypes.c_int64 * 4) * 4), ("coverage", ctypes.c_double * 4),
                ("energy", ctypes.c_double)]


class KmcError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"kmc status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libkmc_b200.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run __graft_entry__.build() (nvcc, sm_100a)")
    L = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, i32, i64, u64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double
    sig = {
        "kmc_create": ([P(KmcGeometry), P(KmcModel), P(KmcDist), P(vp)], i32),
        "kmc_destroy": ([vp], None),
        "kmc_last_error": ([vp], ctypes.c_char_p),
        "kmc_create_error": ([], ctypes.c_char_p),
        "kmc_local_shape": ([vp, P(i64), P(i64), P(i64), P(i64), P(i64)], i32),
        "kmc_set_config": ([vp, vp, i64], i32),
        "kmc_get_config": ([vp, vp, i64], i32),
        "kmc_set_config_device": ([vp, vp, i64], i32),
        "kmc_planes_layout": ([vp, vp, vp, vp, vp], i32),
        "kmc_attach_planes": ([vp, vp, i64], i32),
        "kmc_get_config_device": ([vp, vp, i64], i32),
        "kmc_run": ([vp, dbl, dbl, i32], i32),
        "kmc_substep": ([vp, i32, dbl], i32),
        "kmc_observables": ([vp, P(KmcObs), vp], i32),
        "kmc_get_state": ([vp, P(u64), P(dbl)], i32),
        "kmc_set_state": ([vp, u64, dbl], i32),
        "kmc_rate_table": ([vp, P(i32), vp, vp, vp, vp, vp, P(i32)], i32),
        "kmc_enable_timing": ([vp, i32], i32),
        "kmc_timing": ([vp, P(dbl), P(i64), i32], i32),
        "kmc_partition_plan": ([P(KmcGeometry), i32, i32, i32, vp], i32),
        "kmc_nccl_unique_id": ([vp], i32),
        "kmc_version": ([], ctypes.c_char_p),
        "kmc_vgroup_create": ([P(KmcGeometry), P(KmcModel), i32, i32, vp, vp], i32),
        "kmc_vgroup_run": ([vp, i32, dbl, dbl, i32], i32),
        "kmc_vgroup_sync": ([vp, i32], i32),
        "kmc_set_kernel": ([vp, i32], i32),
        "kmc_correlation": ([vp, i32, i32, vp, vp], i32),
        "kmc_run_multiscale": ([vp, dbl, dbl, i32, i32, u64], i32),
        "kmc_run_nested": ([vp, dbl, dbl, i32, i32, i32, i32], i32),
        "kmc_vgroup_run_nested": ([vp, i32, dbl, dbl, i32, i32, i32, i32], i32),
        "kmc_set_config_packed": ([vp, vp, i64], i32),
        "kmc_get_config_packed": ([vp, vp, i64], i32),
        "kmc_vgroup_create_bounds": ([P(KmcGeometry), P(KmcModel), i32, i32, vp, vp, vp], i32),
        "kmc_workload_mark": ([vp], i32),
        "kmc_workload_partition": ([vp, i32, i32, vp, vp, vp], i32),
        "kmc_vgroup_workload_partition": ([vp, i32, i32, i32, vp, vp, vp], i32),
        "kmc_vgroup_set_fused": ([vp, i32, i32], i32),
        "kmc_abi_sizes": ([vp], None),
        "kmc_record_coverage": ([vp, i32, i64], i32),
        "kmc_stage_config_packed": ([vp, vp, i64], i32),
        "kmc_observables_device": ([vp, vp], i32),
        "kmc_init_random": ([vp, vp, i32, u64], i32),
        "kmc_obs_decode": ([vp, vp, P(KmcObs)], i32),
        "kmc_commit_config": ([vp], i32),
        "kmc_coverage_series": ([vp, vp, i64, P(i64)], i32),
        "kmc_coverage_stats": ([vp, i64, i32, vp, vp, i32, vp], i32),
        "kmc_device_errors": ([vp, P(i32), P(i32)], i32),
        "kmc_vgroup_observables": ([vp, i32, P(KmcObs)], i32),
        "kmc_download_config_packed": ([vp, vp, i64], i32),
        "kmc_download_wait": ([vp], i32),
    }
    ab_build = "KMC_B200_LIB" in os.environ          # an older build under comparison may lack new entry points
    for name, (args, res) in sig.items():
        if ab_build and not hasattr(L, name):
            continue
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def make_geometry(ndim, dims, cell, colours=0, replicas=1, seed=0):
    g = KmcGeometry()
    g.ndim = int(ndim)
    d = list(dims) + [0] * (2 - len(dims))
    c = list(cell) + [0] * (2 - len(cell))
    g.dims[0], g.dims[1] = int(d[0]), int(d[1])
    g.cell[0], g.cell[1] = int(c[0]), int(c[1])
    g.colours = int(colours)
    g.replicas = int(replicas)
    g.seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return g


def make_model(kind="adsdes", ca=1.0, cd=1.0, beta=1.0, K=0.0, h=0.0, c_hop=0.0, k1=0.4, k2=1.0):
    m = KmcModel()
    m.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
    m.ca, m.cd, m.beta, m.K, m.h, m.c_hop, m.k1, m.k2 = (float(v) for v in (ca, cd, beta, K, h, c_hop, k1, k2))
    return m


def partition_plan(ndim, dims, cell, replicas, kind, world, rank):
    """Host-only partition plan (kmc_partition_plan): dict of owned rows / replicas and ring neighbours."""
    g = make_geometry(ndim, dims, cell, replicas=replicas)
    out = (ctypes.c_int64 * 6)()
    st = lib().kmc_partition_plan(ctypes.byref(g), KINDS[kind] if isinstance(kind, str) else int(kind),
                                  int(world), int(rank), out)
    if st != KMC_OK:
        raise KmcError(st, lib().kmc_create_error().decode())
    keys = ["replica_offset", "replicas_local", "row_offset", "rows_local", "rank_up", "rank_down"]
    return dict(zip(keys, [int(v) for v in out]))


def nccl_unique_id() -> bytes:
    buf = (ctypes.c_uint8 * 128)()
    st = lib().kmc_nccl_unique_id(buf)
    if st != KMC_OK:
        raise KmcError(st, lib().kmc_create_error().decode())
    return bytes(buf)


class KMC:
    """One fractional-step KMC context (kmc_create ... kmc_destroy)."""

    def __init__(self, ndim, dims, cell, kind="adsdes", colours=0, replicas=1, seed=0,
                 rank=0, world=1, device=0, stream=None, nccl_id=None, row_bounds=None, fused_exchange=False,
                 **params):
        self._L = lib()
        self.kind = KINDS[kind] if isinstance(kind, str) else int(kind)
        self.nstates = NSTATES[self.kind]
        self.geom = make_geometry(ndim, dims, cell, colours, replicas, seed)
        self.model = make_model(self.kind, **params)
        self.dist = KmcDist()
        self.dist.rank, self.dist.world, self.dist.device = int(rank), int(world), int(device)
        self._id = None
        if nccl_id is not None:
            self._id = (ctypes.c_uint8 * 128).from_buffer_copy(nccl_id)
            self.dist.nccl_unique_id = ctypes.cast(self._id, ctypes.c_void_p)
        self.dist.stream = stream
        self.dist.fused_exchange = 1 if fused_exchange else 0
        self._bounds = None
        if row_bounds is not None:       # caller-chosen slabs (kmc_dist.row_bounds, e.g. from workload_partition)
            self._bounds = np.ascontiguousarray(row_bounds, dtype=np.int64)
            self.dist.row_bounds = self._bounds.ctypes.data
        self._ctx = ctypes.c_void_p()
        st = self._L.kmc_create(ctypes.byref(self.geom), ctypes.byref(self.model), ctypes.byref(self.dist),
                                ctypes.byref(self._ctx))
        if st != KMC_OK:
            raise KmcError(st, self._L.kmc_create_error().decode())
        rl, hl, w, ro, yo = (ctypes.c_int64() for _ in range(5))
        self._check(self._L.kmc_local_shape(self._ctx, ctypes.byref(rl), ctypes.byref(hl), ctypes.byref(w),
                                            ctypes.byref(ro), ctypes.byref(yo)))
        self.local_shape = (rl.value, hl.value, w.value)
        self.replica_offset, self.row_offset = ro.value, yo.value
        self.nbytes = rl.value * hl.value * w.value
        qy, qx = (1, int(cell[0])) if int(ndim) == 1 else (int(cell[0]), int(cell[1]))
        self._strips = int(dims[0]) // qy if int(ndim) == 2 else int(dims[0]) // qx
        # bit-packed layout [plane][cell row][replica][cell column] (kmc_set_config_packed)
        self.packed_shape = (2 if self.nstates == 3 else 1, hl.value // qy, rl.value, w.value // qx)

    def _check(self, st, allow=()):
        if st != KMC_OK and st not in allow:
            raise KmcError(st, self._L.kmc_last_error(self._ctx).decode())
        return st

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            self._L.kmc_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- state -------------------------------------------------------------
    def set_config(self, lat):
        """Host uint8 [replicas_local][rows_local][W] (numpy) -> device (validated, synchronous)."""
        a = np.ascontiguousarray(lat, dtype=np.uint8)
        if a.size != self.nbytes:
            raise ValueError(f"expected {self.nbytes} sites, got {a.size}")
        self._check(self._L.kmc_set_config(self._ctx, a.ctypes.data, a.size))

    def get_config(self):
        out = np.empty(self.local_shape, dtype=np.uint8)
        self._check(self._L.kmc_get_config(self._ctx, out.ctypes.data, out.size))
        return out

    def init_random(self, probs, seed=0):
        """kmc_init_random: i.i.d. site states with probabilities `probs` drawn on the device (R32)."""
        p = np.ascontiguousarray(probs, dtype=np.float64)
        self._check(self._L.kmc_init_random(self._ctx, p.ctypes.data, int(p.size), int(seed) & 0xFFFFFFFFFFFFFFFF))

    def set_config_packed(self, words):
        """Host uint64 words in packed_shape (kmc_set_config_packed: 1 bit per site and plane)."""
        a = np.ascontiguousarray(words, dtype=np.uint64)
        if a.size != int(np.prod(self.packed_shape)):
            raise ValueError(f"expected {int(np.prod(self.packed_shape))} words, got {a.size}")
        self._check(self._L.kmc_set_config_packed(self._ctx, a.ctypes.data, a.size))

    def stage_config_packed(self, words):
        """Pipelined upload (kmc_stage_config_packed): the copy of `words` (packed_shape uint64; pin
        it for a truly asynchronous copy) overlaps the windows in flight; commit_config() makes it
        current.  The array is kept referenced until the commit."""
        a = np.ascontiguousarray(words, dtype=np.uint64)
        if a.size != int(np.prod(self.packed_shape)):
            raise ValueError(f"expected {int(np.prod(self.packed_shape))} words, got {a.size}")
        self._check(self._L.kmc_stage_config_packed(self._ctx, a.ctypes.data, a.size))
        self._staged_host = a

    def commit_config(self):
        try:
            self._check(self._L.kmc_commit_config(self._ctx))
        finally:
            self._staged_host = None

    def get_config_packed(self):
        out = np.empty(self.packed_shape, dtype=np.uint64)
        self._check(self._L.kmc_get_config_packed(self._ctx, out.ctypes.data, out.size))
        return out

    def download_config_packed(self, out):
        """kmc_download_config_packed: asynchronous D2H of the packed lattice into `out` (uint64
        numpy array of packed_shape, ideally pinned); complete after download_wait()."""
        if out.dtype != np.uint64 or out.size != int(np.prod(self.packed_shape)) or not out.flags.c_contiguous:
            raise ValueError(f"need a C-contiguous uint64 array of {int(np.prod(self.packed_shape))} words")
        self._check(self._L.kmc_download_config_packed(self._ctx, out.ctypes.data, out.size))
        self._download_host = out

    def download_wait(self):
        try:
            self._check(self._L.kmc_download_wait(self._ctx))
        finally:
            self._download_host = None

    # ---- f4: workload histogram and cdf re-partition -----------------------------
    def workload_mark(self):
        """kmc_workload_mark: the workload interval starts now."""
        self._check(self._L.kmc_workload_mark(self._ctx))

    def workload_partition(self, parts, granule=1):
        """kmc_workload_partition: strip loads since the mark and their cdf split into `parts`."""
        return _partition(self._L, self._check, self._L.kmc_workload_partition, self._ctx, parts, granule,
                          self._strips)

    def set_config_device(self, ptr, nbytes):
        """Device uint8 buffer (e.g. torch CUDA tensor .data_ptr()), stream-ordered."""
        self._check(self._L.kmc_set_config_device(self._ctx, ctypes.c_void_p(ptr), int(nbytes)))

    def get_config_device(self, ptr, nbytes):
        self._check(self._L.kmc_get_config_device(self._ctx, ctypes.c_void_p(ptr), int(nbytes)))

    def planes_layout(self):
        """kmc_planes_layout: {'planes', 'words_per_plane', 'storage_rows', 'ghost'} of the working lattice."""
        n, w, r, gh = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int32()
        self._check(self._L.kmc_planes_layout(self._ctx, ctypes.byref(n), ctypes.byref(w), ctypes.byref(r),
                                              ctypes.byref(gh)))
        return {"planes": n.value, "words_per_plane": w.value, "storage_rows": r.value, "ghost": gh.value}

    def attach_planes(self, ptr, nwords):
        """kmc_attach_planes: run on the caller's device buffer (e.g. a torch int64 CUDA tensor's
        data_ptr(), kept alive by the caller until close) as the working lattice."""
        self._check(self._L.kmc_attach_planes(self._ctx, ctypes.c_void_p(ptr), int(nwords)))

    # ---- the hot path --------------------------------------------------------
    def run(self, T, dt, scheme="lie"):
        """kmc_run; returns True if the last macro-step was shortened (KMC_WTRUNCATED)."""
        sc = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        st = self._check(self._L.kmc_run(self._ctx, float(T), float(dt), sc), allow=(KMC_WTRUNCATED,))
        return st == KMC_WTRUNCATED

    def run_multiscale(self, T, dt, n_fast, inner="lie", fast_classes=0):
        """kmc_run_multiscale (eq.(strang3)): e^{dt/2 L_slow} [e^{dt/n L_fast}]^n e^{dt/2 L_slow}
        per macro-step, each factor split over colours with `inner`; returns the truncation flag."""
        sc = SCHEMES[inner] if isinstance(inner, str) else int(inner)
        st = self._check(self._L.kmc_run_multiscale(self._ctx, float(T), float(dt), int(n_fast), sc,
                                                    int(fast_classes)), allow=(KMC_WTRUNCATED,))
        return st == KMC_WTRUNCATED

    def run_nested(self, T, dt, n_inner, outer="lie", inner="lie", block=2):
        """kmc_run_nested (f3, eq.(opdecomp2), R28): outer Lie/Strang over the two outer block
        colours, each outer factor n_inner cycles of `inner` over the cell colours; returns the
        truncation flag."""
        so = SCHEMES[outer] if isinstance(outer, str) else int(outer)
        si = SCHEMES[inner] if isinstance(inner, str) else int(inner)
        st = self._check(self._L.kmc_run_nested(self._ctx, float(T), float(dt), int(n_inner), so, si,
                                                int(block)), allow=(KMC_WTRUNCATED,))
        return st == KMC_WTRUNCATED

    def substep(self, colour, duration):
        self._check(self._L.kmc_substep(self._ctx, int(colour), float(duration)))

    def observables(self, per_cell=False):
        o = KmcObs()
        cells = None
        ptr = None
        if per_cell:
            R, H, W = self.local_shape
            qy = 1 if self.geom.ndim == 1 else self.geom.cell[0]
            qx = self.geom.cell[0] if self.geom.ndim == 1 else self.geom.cell[1]
            cells = np.zeros((R, H // qy, W // qx), dtype=np.uint32)
            ptr = cells.ctypes.data
        self._check(self._L.kmc_observables(self._ctx, ctypes.byref(o), ptr))
        d = self._obs_dict(o)
        if per_cell:
            d["per_cell_events"] = cells
        return d

    @staticmethod
    def _obs_dict(o):
        return {
            "time": o.time, "windows": int(o.windows), "events": int(o.events),
            "n_state": np.array(o.n_state[:], dtype=np.int64),
            "nn_pairs": np.array([o.nn_pairs[i][:] for i in range(4)], dtype=np.int64),
            "n_state_by_colour": np.array([o.n_state_by_colour[i][:] for i in range(4)], dtype=np.int64),
            "coverage": np.array(o.coverage[:]), "energy": o.energy,
        }

    def observables_device(self, dev_ptr):
        """kmc_observables_device: enqueue the a8 counters of the current state into OBS_WORDS
        uint64 at device address dev_ptr (e.g. a torch int64 tensor's data_ptr()); no host sync."""
        self._check(self._L.kmc_observables_device(self._ctx, ctypes.c_void_p(int(dev_ptr))))

    def obs_decode(self, words):
        """kmc_obs_decode of a host copy of the OBS_WORDS counters: the observables() dict."""
        a = np.ascontiguousarray(words)
        if a.dtype != np.uint64:
            a = a.astype(np.int64).view(np.uint64)
        o = KmcObs()
        self._check(self._L.kmc_obs_decode(self._ctx, a.ctypes.data, ctypes.byref(o)))
        return self._obs_dict(o)

    def correlation(self, rmax, state=1):
        """Two-point correlation counts (kmc_correlation): {'x': int64[rmax+1], 'y': int64[rmax+1]},
        pairs (x, x + r e) with both sites in `state`, summed over the lattice."""
        ox = np.zeros(int(rmax) + 1, dtype=np.int64)
        oy = np.zeros(int(rmax) + 1, dtype=np.int64)
        self._check(self._L.kmc_correlation(self._ctx, int(rmax), int(state), ox.ctypes.data, oy.ctypes.data))
        return {"x": ox, "y": oy}

    def record_coverage(self, capacity, state=1):
        """Start recording the coverage process (kmc_record_coverage): sample 0 now, then one per
        macro-step of run / run_multiscale / run_nested (capacity 0 stops and frees)."""
        self._check(self._L.kmc_record_coverage(self._ctx, int(state), int(capacity)))

    def coverage_series(self):
        """Recorded samples (kmc_coverage_series): int64 [n][local replicas] site counts."""
        n = ctypes.c_int64()
        self._check(self._L.kmc_coverage_series(self._ctx, None, 0, ctypes.byref(n)))
        out = np.zeros((int(n.value), self.local_shape[0]), dtype=np.int64)
        if out.size:
            self._check(self._L.kmc_coverage_series(self._ctx, out.ctypes.data, out.shape[0], ctypes.byref(n)))
        return out

    def coverage_stats(self, max_lag, first=0, bins=0):
        """kmc_coverage_stats over samples [first, n): {'mean', 'var' (= gamma(0)), 'acf'
        float64[max_lag+1], 'hist' int64[bins] (bins > 0)}."""
        acf = np.zeros(int(max_lag) + 1, dtype=np.float64)
        mom = np.zeros(2, dtype=np.float64)
        hist = np.zeros(int(bins), dtype=np.int64) if bins else None
        self._check(self._L.kmc_coverage_stats(self._ctx, int(first), int(max_lag), acf.ctypes.data, mom.ctypes.data,
                                               int(bins), hist.ctypes.data if bins else None))
        return {"mean": float(mom[0]), "var": float(mom[1]), "acf": acf, "hist": hist}

    def device_errors(self):
        """kmc_device_errors: {'bad_spins': last set_config_device clamped out-of-range spins,
        'wait_timeouts': a fused-exchange flag wait gave up} (synchronises)."""
        b, t = ctypes.c_int32(), ctypes.c_int32()
        self._check(self._L.kmc_device_errors(self._ctx, ctypes.byref(b), ctypes.byref(t)))
        return {"bad_spins": bool(b.value), "wait_timeouts": bool(t.value)}

    def get_state(self):
        w, t = ctypes.c_uint64(), ctypes.c_double()
        self._check(self._L.kmc_get_state(self._ctx, ctypes.byref(w), ctypes.byref(t)))
        return int(w.value), float(t.value)

    def set_state(self, windows, time):
        self._check(self._L.kmc_set_state(self._ctx, int(windows), float(time)))

    def rate_table(self):
        n, F = ctypes.c_int32(), ctypes.c_int32()
        ty = (ctypes.c_int32 * 32)(); di = (ctypes.c_int32 * 32)(); ka = (ctypes.c_int32 * 32)()
        ra = (ctypes.c_double * 32)(); ru = (ctypes.c_uint64 * 32)()
        self._check(self._L.kmc_rate_table(self._ctx, ctypes.byref(n), ty, di, ka, ra, ru, ctypes.byref(F)))
        k = n.value
        return {"n": k, "type": np.array(ty[:k]), "dir": np.array(di[:k]), "kappa": np.array(ka[:k]),
                "rate": np.array(ra[:k]), "rate_u64": np.array(ru[:k], dtype=np.uint64), "F": F.value}

    def set_kernel(self, mode="auto"):
        """Window-kernel choice: 'auto', 'queue' (lane-per-cell, global closure loads) or 'tile'
        (2D spin flip: shared-memory tiles).  Performance only; results are bit-identical."""
        self._check(self._L.kmc_set_kernel(self._ctx, KERNELS[mode] if isinstance(mode, str) else int(mode)))

    # ---- timing (bench) --------------------------------------------------------
    def enable_timing(self, on=True):
        self._check(self._L.kmc_enable_timing(self._ctx, 1 if on else 0))

    def timing(self, reset=True):
        ms, n = ctypes.c_double(), ctypes.c_int64()
        self._check(self._L.kmc_timing(self._ctx, ctypes.byref(ms), ctypes.byref(n), 1 if reset else 0))
        return ms.value, n.value


class _Rank(KMC):
    """One virtual rank of a VGroup (created by kmc_vgroup_create, not kmc_create)."""

    def __init__(self, L, ctx, kind, geom, model):
        self._L = L
        self._ctx = ctx
        self.kind = kind
        self.nstates = NSTATES[kind]
        self.geom = geom
        self.model = model
        rl, hl, w, ro, yo = (ctypes.c_int64() for _ in range(5))
        self._check(L.kmc_local_shape(ctx, ctypes.byref(rl), ctypes.byref(hl), ctypes.byref(w),
                                      ctypes.byref(ro), ctypes.byref(yo)))
        self.local_shape = (rl.value, hl.value, w.value)
        self.replica_offset, self.row_offset = ro.value, yo.value
        self.nbytes = rl.value * hl.value * w.value
        qy, qx = (1, int(geom.cell[0])) if int(geom.ndim) == 1 else (int(geom.cell[0]), int(geom.cell[1]))
        self.packed_shape = (2 if self.nstates == 3 else 1, hl.value // qy, rl.value, w.value // qx)


def _partition(L, check, fn, ctx, parts, granule, nstrips):
    bounds = np.zeros(int(parts) + 1, dtype=np.int64)
    loads = np.zeros(nstrips, dtype=np.uint64)
    imb = np.zeros(2, dtype=np.float64)
    check(fn(ctx, int(parts), int(granule), bounds.ctypes.data, loads.ctypes.data, imb.ctypes.data))
    return {"bounds": bounds, "strip_load": loads, "imbalance": float(imb[0]), "imbalance_even": float(imb[1])}


class VGroup:
    """`world` virtual ranks of one 2D lattice on one GPU (kmc_vgroup_*): the multi-GPU slab
    decomposition and halo-exchange protocol, with stream-ordered copies instead of NCCL."""

    def __init__(self, world, dims, cell, kind="adsdes", colours=0, replicas=1, seed=0, device=0,
                 stream=None, row_bounds=None, **params):
        L = lib()
        self._L = L
        self.world = int(world)
        k = KINDS[kind] if isinstance(kind, str) else int(kind)
        self.geom = make_geometry(2, dims, cell, colours, replicas, seed)
        self.model = make_model(k, **params)
        arr = (ctypes.c_void_p * self.world)()
        self._bounds = None if row_bounds is None else np.ascontiguousarray(row_bounds, dtype=np.int64)
        st = L.kmc_vgroup_create_bounds(ctypes.byref(self.geom), ctypes.byref(self.model), self.world, int(device),
                                        stream, None if self._bounds is None else self._bounds.ctypes.data, arr)
        self._strips = int(dims[0]) // int(cell[0])
        if st != KMC_OK:
            raise KmcError(st, L.kmc_create_error().decode())
        self._arr = arr
        self.ranks = [_Rank(L, ctypes.c_void_p(arr[r]), k, self.geom, self.model) for r in range(self.world)]

    def _check(self, st, allow=()):
        if st != KMC_OK and st not in allow:
            raise KmcError(st, self._L.kmc_last_error(self.ranks[0]._ctx).decode())
        return st

    def set_config(self, lat):
        """Full lattice [replicas][H][W] -> each rank's slab."""
        lat = np.ascontiguousarray(lat, dtype=np.uint8)
        for rk in self.ranks:
            h = rk.local_shape[1]
            rk.set_config(lat[:, rk.row_offset:rk.row_offset + h])

    def get_config(self):
        return np.concatenate([rk.get_config() for rk in self.ranks], axis=1)

    def run(self, T, dt, scheme="lie"):
        sc = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        return self._check(self._L.kmc_vgroup_run(self._arr, self.world, float(T), float(dt), sc),
                           allow=(KMC_WTRUNCATED,)) == KMC_WTRUNCATED

    def run_nested(self, T, dt, n_inner, outer="lie", inner="lie", block=2):
        so = SCHEMES[outer] if isinstance(outer, str) else int(outer)
        si = SCHEMES[inner] if isinstance(inner, str) else int(inner)
        return self._check(self._L.kmc_vgroup_run_nested(self._arr, self.world, float(T), float(dt), int(n_inner),
                                                         so, si, int(block)),
                           allow=(KMC_WTRUNCATED,)) == KMC_WTRUNCATED

    def set_fused(self, enable=True):
        """kmc_vgroup_set_fused: the halo exchange folded into the window kernels (peer writes)."""
        self._check(self._L.kmc_vgroup_set_fused(self._arr, self.world, int(bool(enable))))

    def workload_mark(self):
        for rk in self.ranks:
            self._check(self._L.kmc_workload_mark(rk._ctx))

    def workload_partition(self, parts, granule=1):
        fn = lambda arr, *rest: self._L.kmc_vgroup_workload_partition(arr, self.world, *rest)
        return _partition(self._L, self._check, fn, self._arr, parts, granule, self._strips)

    def observables(self):
        """kmc_vgroup_observables: the group's observables (counters summed over the ranks in C)."""
        o = KmcObs()
        self._check(self._L.kmc_vgroup_observables(self._arr, self.world, ctypes.byref(o)))
        return KMC._obs_dict(o)

    def close(self):
        for rk in self.ranks:
            rk.close()
