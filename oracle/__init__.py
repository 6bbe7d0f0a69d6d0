"""CPU oracles for the fractional-step KMC hot path (arXiv:1105.4673).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  It shares no code with ``paper_1105_4673_b200`` (the CUDA product
path) and neither imports the other.

Modules
  fskmc      O2 -- serial fractional-step oracle (bit-exact reference), the
             schedule of eq.(lie)/eq.(strang)/eq.(SLPCS) in plain Python
             driving the C per-window loop of ``fskmc_oracle.c``.
  ssa        O1 -- exact serial SSA (statistical reference).
  bruteforce dense master-equation generators on <= 12 sites (P4-P6 pins).
  exact      closed forms: non-interacting two-state law, 1D transfer
             matrix, the paper's eq.(exactcov1d) and eq.(exactcov2d).

Parity status per function is listed in DESIGN.md §5 ("pins").
"""
import ctypes
import os

import numpy as np

from . import _build

_lib = None


def lib():
    """Load (building if needed) the oracle's C library."""
    global _lib
    if _lib is None:
        path = _build.build()
        L = ctypes.CDLL(path)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_philox4x32_10.restype = None
        L.orc_log.argtypes = [ctypes.c_double]
        L.orc_log.restype = ctypes.c_double
        ip = ctypes.POINTER(ctypes.c_int)
        dp = ctypes.POINTER(ctypes.c_double)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.orc_classes.argtypes = [ctypes.c_int, ctypes.c_int, dp, ip, ip, ip, dp]
        L.orc_classes.restype = ctypes.c_int
        L.orc_types_per_site.argtypes = [ctypes.c_int, ctypes.c_int]
        L.orc_types_per_site.restype = ctypes.c_int
        L.orc_quantise.argtypes = [dp, ctypes.c_int, ctypes.c_int, ctypes.c_int, u64p]
        L.orc_quantise.restype = ctypes.c_int
        L.orc_cell_colour.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        L.orc_cell_colour.restype = ctypes.c_int
        L.orc_window.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                 ctypes.c_int, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                 ctypes.c_int, ip, ip, ip, u64p, ctypes.c_int, ctypes.c_void_p]
        L.orc_window.restype = ctypes.c_int64
        L.orc_window_cells.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                       ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                       ctypes.c_int64, ctypes.c_double, ctypes.c_uint64, ctypes.c_uint64,
                                       ctypes.c_int, ip, ip, ip, u64p, ctypes.c_int, ctypes.c_void_p]
        L.orc_window_cells.restype = ctypes.c_int64
        L.orc_ssa.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                              ctypes.c_int, ip, ip, ip, u64p, ctypes.c_int, ctypes.c_uint64,
                              ctypes.c_uint32, dp, ctypes.c_int, ctypes.c_void_p]
        L.orc_ssa.restype = ctypes.c_int64
        _lib = L
    return _lib


def philox4x32_10(ctr, key):
    """Philox4x32-10 of one 128-bit counter under a 64-bit key (Random123 convention)."""
    c = (ctypes.c_uint32 * 4)(*[int(v) & 0xFFFFFFFF for v in ctr])
    k = (ctypes.c_uint32 * 2)(*[int(v) & 0xFFFFFFFF for v in key])
    o = (ctypes.c_uint32 * 4)()
    lib().orc_philox4x32_10(c, k, o)
    return tuple(int(v) for v in o)


def log_spec(x: float) -> float:
    """The specified natural log: the table-driven FMA sequence of DESIGN.md §3.1 (reading R26)."""
    return lib().orc_log(float(x))
