"""O1 -- exact serial SSA on the whole lattice (statistical reference).

TEST INFRASTRUCTURE (see oracle/__init__.py).  The CTMC of eq.(generator)
 simulated directly: exponential clock with the total rate
eq.(totalrate) and rate-proportional selection eq.(skeleton)
 over every slot of the lattice (Fenwick tree, u64 fixed-point
rates of the same class list as O2).  RNG stream: Philox tag 3, disjoint
from O2's tag 0.
"""
import ctypes

import numpy as np

from . import lib
from .fskmc import KIND, rate_table


def ssa_snapshots(lat2d, ndim, kind, params, T_obs, seed=0, stream=0):
    """Run one replica from ``lat2d`` ([H][W] uint8, H=1 in 1D); return the lattice
    at each time in ``T_obs`` (sorted) as an array [len(T_obs)][H][W], and the
    number of events executed."""
    kind = KIND[kind] if isinstance(kind, str) else int(kind)
    lat = np.ascontiguousarray(lat2d, dtype=np.uint8).copy()
    H, W = lat.shape
    tab = rate_table(kind, ndim, params, H * W)  # lambda <= 2^62 over the whole lattice
    T = np.ascontiguousarray(np.asarray(T_obs, dtype=np.float64))
    out = np.zeros((len(T), H, W), dtype=np.uint8)
    ip = ctypes.POINTER(ctypes.c_int)
    nev = lib().orc_ssa(lat.ctypes.data, H, W, ndim, tab["n"],
                        tab["type"].ctypes.data_as(ip), tab["dir"].ctypes.data_as(ip),
                        tab["kappa"].ctypes.data_as(ip),
                        tab["rate_u64"].ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)),
                        tab["F"], int(seed), int(stream),
                        T.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(T), out.ctypes.data)
    if nev < 0:
        raise MemoryError("orc_ssa allocation failed")
    return out, int(nev)
