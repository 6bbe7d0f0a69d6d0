"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

Holds none of the method's arithmetic: it only draws initial lattices and
parameter sets ("input recipe").  Both the CUDA path (through
kmc_set_config) and the oracle receive the same uint8 arrays from here.
"""
import numpy as np

SEED_BASE = 0x5EED0001


def bernoulli_lattice(shape, p=0.5, seed=SEED_BASE, chunk=1 << 24):
    """Sites occupied (state 1) independently with probability p; uint8 site-major.
    Drawn in chunks of `chunk` sites (float32 uniforms) so 32768^2 lattices fit in memory."""
    rng = np.random.default_rng(seed)
    out = np.empty(int(np.prod(shape)), dtype=np.uint8)
    p32 = np.float32(p)
    for i in range(0, out.size, chunk):
        n = min(chunk, out.size - i)
        out[i:i + n] = rng.random(n, dtype=np.float32) < p32
    return out.reshape(shape)


def categorical_lattice(shape, probs, seed=SEED_BASE):
    """Sites in state s with probability probs[s] (ZGB: 0 vacant, 1 CO, 2 O)."""
    rng = np.random.default_rng(seed)
    cum = np.cumsum(np.asarray(probs, dtype=np.float64))[:-1].astype(np.float32)
    out = np.empty(int(np.prod(shape)), dtype=np.uint8)
    chunk = 1 << 24
    for i in range(0, out.size, chunk):
        n = min(chunk, out.size - i)
        out[i:i + n] = np.searchsorted(cum, rng.random(n, dtype=np.float32), side="right")
    return out.reshape(shape)


def colour_full_lattice(shape, ndim, cell, C, colour=1):
    """R#/P5 asymmetric start: sites of cells with the given colour full, others empty."""
    R, H, W = shape
    if ndim == 1:
        qy, qx = 1, cell[0]
    else:
        qy, qx = cell
    cy = np.arange(H)[:, None] // qy
    cx = np.arange(W)[None, :] // qx
    if C == 2:
        col = (cx & 1) if ndim == 1 else ((cx + cy) & 1)
    else:
        col = (cx & 1) + 2 * (cy & 1)
    col = np.broadcast_to(col, (H, W))
    return np.broadcast_to((col == colour).astype(np.uint8), shape).copy()


def packed_lattice(lat, ndim, cell, nplanes):
    """The same input in the library's bit-packed upload format (kmc_set_config_packed, layout
    [plane][cell row][replica][cell column], bit ly*q_x + lx of a word = site (ly, lx) of the cell,
    plane p = (site == p + 1)).  Layout conversion only; q_x must be a multiple of 8."""
    R, H, W = lat.shape
    qy, qx = (1, cell[0]) if ndim == 1 else cell
    if qx % 8 or qx * qy > 64:
        raise ValueError("packed_lattice needs q_x % 8 == 0 and q_x*q_y <= 64")
    My, Mx, nb = H // qy, W // qx, qx * qy // 8
    out = np.zeros((nplanes, My, R, Mx, 8), dtype=np.uint8)
    for p in range(nplanes):
        b = np.packbits(lat == p + 1, axis=2, bitorder="little")          # [R][H][W/8]
        b = b.reshape(R, My, qy, Mx, qx // 8).transpose(1, 0, 3, 2, 4).reshape(My, R, Mx, nb)
        out[p, ..., :nb] = b
    return out.view(np.uint64).reshape(nplanes, My, R, Mx)


# Named workloads.
WORKLOADS = {
    # target / bench N=1: 2D Ising ads/des 32768^2, 8x8 cells, Lie dt=1,
    # K=1, ca=cd=1, beta=1.5, h_dyn=-2 (paper's h=2 zero-field point), Bernoulli(1/2)
    "ising2d_32768": dict(ndim=2, dims=(32768, 32768), cell=(8, 8), kind="adsdes",
                          params=dict(ca=1.0, cd=1.0, beta=1.5, K=1.0, h=-2.0),
                          scheme="lie", dt=1.0, init=0.5),
    # the same lattice and model with the Strang splitting (the bench default: at the paper's dt = 1
    # it meets the north star's |dtheta| <= 1e-2 accuracy bar, tests/test_gpu_statistics.py)
    "ising2d_32768_strang": dict(ndim=2, dims=(32768, 32768), cell=(8, 8), kind="adsdes",
                                 params=dict(ca=1.0, cd=1.0, beta=1.5, K=1.0, h=-2.0),
                                 scheme="strang", dt=1.0, init=0.5),
    "ising2d_1024": dict(ndim=2, dims=(1024, 1024), cell=(8, 8), kind="adsdes",
                         params=dict(ca=1.0, cd=1.0, beta=1.5, K=1.0, h=-2.0),
                         scheme="lie", dt=1.0, init=0.5),
    "ising1d_65536": dict(ndim=1, dims=(65536,), cell=(32,), kind="adsdes",
                          params=dict(ca=1.0, cd=1.0, beta=2.0, K=1.0, h=0.0),
                          scheme="lie", dt=1.0, init=0.0),
    # cfg2 as SURVEY §8(d) runs it: 64 independent replicas per GPU (the paper averages over
    # M = 1000 realisations)
    "ising1d_65536x64": dict(ndim=1, dims=(65536,), cell=(32,), kind="adsdes",
                             params=dict(ca=1.0, cd=1.0, beta=2.0, K=1.0, h=0.0),
                             scheme="lie", dt=1.0, init=0.0, replicas_per_gpu=64),
    # cfg1: non-interacting 1D, N = 1024, Q = 32, M = 1000 replicas per GPU, Lie dt = 0.1
    "noninteracting1d_1024x1000": dict(ndim=1, dims=(1024,), cell=(32,), kind="adsdes",
                                       params=dict(ca=1.0, cd=0.5, beta=1.0, K=0.0, h=0.0),
                                       scheme="lie", dt=0.1, init=0.0, replicas_per_gpu=1000),
    "diff2d_8192": dict(ndim=2, dims=(8192, 8192), cell=(8, 8), kind="adsdes_diff",
                        params=dict(ca=1.0, cd=1.0, beta=1.5, K=1.0, h=-2.0, c_hop=1.0),
                        scheme="strang", dt=1.0, init=0.5),
    "zgb2d_32768": dict(ndim=2, dims=(32768, 32768), cell=(8, 8), kind="zgb",
                        params=dict(k1=0.4, k2=1.0),
                        scheme="lie", dt=0.1, init=0.0),
    # cfg5 as BASELINE names it: adsorption / desorption / diffusion / reaction (ZGB + CO hops)
    "zgbdiff2d_32768": dict(ndim=2, dims=(32768, 32768), cell=(8, 8), kind="zgb_diff",
                            params=dict(k1=0.4, k2=1.0, c_hop=1.0),
                            scheme="lie", dt=0.1, init=0.0),
    # ZGB with the fast O diffusion of P:1211-1213 (R33)
    "zgbodiff2d_32768": dict(ndim=2, dims=(32768, 32768), cell=(8, 8), kind="zgb_odiff",
                             params=dict(k1=0.4, k2=1.0, c_hop=1.0),
                             scheme="lie", dt=0.1, init=0.0),
}
