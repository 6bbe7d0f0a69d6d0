"""f4 -- workload histogram and the cdf ("mass transport") re-partition of PAPER.md §Mass
Transport and Dynamic Workload Balancing, reading R29 of DESIGN.md.

TEST INFRASTRUCTURE (see oracle/__init__.py): plain numpy, written from the paper, shares no code
with the CUDA path.

  eq.(wload) P:890-896   W(m) = # jumps in cell C_m during the interval (per-cell event counts)
  P:919-925              map the cdf of W onto the uniform distribution over P processors:
                         processor l gets the mass in [(l-1)/P, l/P) of the cdf
  P:936-938              in 2D the re-balancing stays one-dimensional with strips: a strip =
                         one row of cells (all columns and replicas); 1D: a strip = one cell
"""
import numpy as np


def strip_loads(W, ndim):
    """Per-strip workload from per-cell counts W[replica][cell row][cell column] (uint)."""
    W = np.asarray(W, dtype=np.uint64)
    if ndim == 2:
        return W.sum(axis=(0, 2), dtype=np.uint64)
    return W.sum(axis=(0, 1), dtype=np.uint64)


def cdf_bounds(loads, parts, granule=1):
    """R29: strip bounds b_0 = 0 < b_1 < ... < b_P = M of the P groups.

    b_l = min{ s + 1 : P * (w_0 + ... + w_s) >= l * S }    (S = total; the cdf reaches l/P)
    then rounded to the nearest multiple of `granule` (ties up), and clamped so that every group
    keeps at least one granule: b_l in [b_{l-1} + g, M - (P - l) g].  S = 0: the even split
    b_l = round(l M / P).  Exact integer arithmetic."""
    w = [int(x) for x in loads]
    M, P, g = len(w), int(parts), int(granule)
    if P < 1 or g < 1 or M % g or M < P * g:
        raise ValueError("need M a multiple of granule and M >= parts * granule")
    S = sum(w)
    raw = []
    for l in range(1, P):
        if S == 0:
            raw.append((l * M + P // 2) // P)
            continue
        cum = 0
        for s in range(M):
            cum += w[s]
            if P * cum >= l * S:
                raw.append(s + 1)
                break
    b = [0]
    for l, x in enumerate(raw, start=1):
        r = g * ((2 * x + g) // (2 * g))
        r = max(r, b[-1] + g)
        r = min(r, M - (P - l) * g)
        b.append(r)
    b.append(M)
    return np.array(b, dtype=np.int64)


def group_loads(loads, bounds):
    w = np.asarray(loads, dtype=np.uint64)
    return np.array([int(w[bounds[i]:bounds[i + 1]].sum()) for i in range(len(bounds) - 1)], dtype=np.int64)


def imbalance(loads, bounds):
    """max group load / mean group load (1 = perfectly balanced; S = 0 gives 1)."""
    gl = group_loads(loads, bounds)
    S = int(gl.sum())
    if S == 0:
        return 1.0
    return float(gl.max()) * len(gl) / S


def even_bounds(M, parts, granule=1):
    return cdf_bounds(np.zeros(M, dtype=np.uint64), parts, granule)
