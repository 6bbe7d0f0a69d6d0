"""Pins of the O2 (fractional-step) and O1 (exact SSA) oracles against the
brute-force laws and the closed forms (CPU, statistical).

Tolerances: Monte Carlo means are compared within Z = 4.5 standard errors
(per comparison family false-alarm rate < 1e-4), computed from the exact
law's own variance.
"""
import math

import numpy as np
import pytest

from oracle import bruteforce as bf
from oracle import exact
from oracle.fskmc import FSKMC, model_params
from oracle.ssa import ssa_snapshots

Z = 4.5

MODELS_1D = {
    "adsdes": dict(ca=1.0, cd=1.0, beta=1.0, K=1.0, h=-1.0),
    "adsdes_diff": dict(ca=0.5, cd=1.0, beta=1.0, K=1.0, h=-1.0, c_hop=1.3),
    "zgb": dict(k1=0.4, k2=1.0),
    "zgb_diff": dict(k1=0.4, k2=1.0, c_hop=0.8),
    "zgb_odiff": dict(k1=0.4, k2=1.0, c_hop=0.9),    # fast O diffusion (R33)
}


def bf_model(kind, p):
    m = dict(kind=kind, ca=0.0, cd=0.0, beta=0.0, K=0.0, h=0.0, c_hop=0.0, k1=0.4, k2=1.0)
    m.update(p)
    return m


def confs_index(lat_batch, S):
    """Configuration index sum_i sigma_i S^i (sites row-major) for each replica."""
    R = lat_batch.shape[0]
    flat = lat_batch.reshape(R, -1).astype(np.int64)
    pw = S ** np.arange(flat.shape[1], dtype=np.int64)
    return flat @ pw


def check_law(samples_idx, p, Z=Z):
    """Each state's empirical frequency within Z binomial SE of the exact law p
    (plus a small absolute floor for states with p ~ 0)."""
    R = len(samples_idx)
    emp = np.bincount(samples_idx, minlength=len(p)) / R
    se = np.sqrt(p * (1 - p) / R)
    bad = np.abs(emp - p) > Z * se + 3.0 / R
    assert not bad.any(), (np.nonzero(bad)[0][:5], emp[bad][:5], p[bad][:5])


@pytest.mark.parametrize("kind", list(MODELS_1D))
def test_o2_one_window_law_1d(kind):
    """One window of colour 0 samples e^{D Q^0} exactly (eq.(exact), R5)."""
    N, q, D, R = 4, 2, 0.8, 30000
    p = MODELS_1D[kind]
    lat = bf.Lattice(1, 1, N, 1, q, 2)
    Q, Qc, S = bf.generators(bf_model(kind, p), lat)
    start = [1, 0, 0, 2 if S == 3 else 1]
    p0 = bf.point_mass(S, N, start)
    law = bf.evolve(p0, Qc[0], D)
    sim = FSKMC(1, (N,), (q,), kind, model_params(**p), colours=2, replicas=R, seed=11)
    sim.set_config(np.broadcast_to(np.array(start, np.uint8), (R, 1, N)))
    sim.substep(0, D)
    check_law(confs_index(sim.get_config(), S), law)


def test_o2_one_window_law_2d_diffusion_4colour():
    """2D 4x4 torus, 2x2 cells, 4 colours (R6), ads/des + hops: mean site occupancies
    after one window of colour 3 match e^{D Q^3}."""
    kind = "adsdes_diff"
    p = dict(ca=0.6, cd=1.0, beta=1.0, K=0.7, h=-1.0, c_hop=1.5)
    lat = bf.Lattice(2, 4, 4, 2, 2, 4)
    Q, Qc, S = bf.generators(bf_model(kind, p), lat)
    rng = np.random.default_rng(3)
    start = rng.integers(0, 2, 16)
    law = bf.evolve(bf.point_mass(S, 16, start), Qc[3], 0.9)
    confs = np.array(np.unravel_index(np.arange(S ** 16), [S] * 16))[::-1].T  # digit i = site i
    mean_exact = law @ confs
    var_exact = law @ (confs ** 2) - mean_exact ** 2
    R = 20000
    sim = FSKMC(2, (4, 4), (2, 2), kind, model_params(**p), colours=4, replicas=R, seed=5)
    sim.set_config(np.broadcast_to(start.reshape(1, 4, 4).astype(np.uint8), (R, 4, 4)))
    sim.substep(3, 0.9)
    emp = sim.get_config().reshape(R, 16).mean(axis=0)
    assert np.all(np.abs(emp - mean_exact) <= Z * np.sqrt(var_exact / R) + 1e-3)


@pytest.mark.parametrize("scheme", ["lie", "strang", "random"])
def test_o2_scheme_law_1d(scheme):
    """Mean coverage of each scheme after T = 2 equals the brute-force law of
    eq.(lie)/eq.(strang)/eq.(SL) (random: xi-averaged), asymmetric start (R#-P5)."""
    N, q, dt, T, R = 8, 2, 0.5, 2.0, 20000
    p = dict(ca=1.0, cd=1.0, beta=1.0, K=1.0, h=-1.0)
    lat = bf.Lattice(1, 1, N, 1, q, 2)
    Q, Qc, S = bf.generators(bf_model("adsdes", p), lat)
    start = np.array([1 if lat.colour(i) == 1 else 0 for i in range(N)], np.uint8)
    if scheme == "random":   # the realised schedule is shared by all replicas (R4)
        from oracle.fskmc import substeps, RANDOM
        seq = [cd for w in range(0, int(round(T / dt)) * 2, 2) for cd in substeps(RANDOM, 2, dt, 21, w)]
        law = bf.law_sequence(bf.point_mass(S, N, start), Qc, seq)
    else:
        law = bf.law(bf.point_mass(S, N, start), Q, Qc, scheme, dt, T, 2)
    cov = bf.coverage_values(lat, S)
    m, v = law @ cov, law @ cov ** 2 - (law @ cov) ** 2
    sim = FSKMC(1, (N,), (q,), "adsdes", model_params(**p), colours=2, replicas=R, seed=21)
    sim.set_config(np.broadcast_to(start, (R, 1, N)))
    sim.run(T, dt, scheme)
    emp = sim.get_config().reshape(R, N).mean(axis=1)
    assert abs(emp.mean() - m) <= Z * math.sqrt(v / R)


def test_o2_noninteracting_closed_form_mean_and_variance():
    """cfg1 shape: K = 0, N = 1024, Q = 32, Lie, T = 1 and 10: coverage is
    Binomial(N R, theta(t)) -- mean and variance pinned."""
    R, N = 8, 1024
    p = dict(ca=1.0, cd=0.5, beta=1.0, K=0.0, h=0.0)
    sim = FSKMC(1, (N,), (32,), "adsdes", model_params(**p), colours=2, replicas=R, seed=3)
    sim.run(1.0, 0.1, "lie")
    th = exact.noninteracting_theta(1.0, 1.0, 0.5)
    lat = sim.get_config().reshape(R, N)
    n = R * N
    assert abs(lat.mean() - th) <= Z * math.sqrt(th * (1 - th) / n)
    per_rep = lat.mean(axis=1)   # variance of per-replica coverage = th(1-th)/N
    assert 0.2 < per_rep.var(ddof=1) / (th * (1 - th) / N) < 3.5
    sim.run(9.0, 1.0, "lie")
    th10 = exact.noninteracting_theta(10.0, 1.0, 0.5)
    assert abs(sim.get_config().mean() - th10) <= Z * math.sqrt(th10 * (1 - th10) / n)


def test_o2_gibbs_equilibrium_1d_transfer_matrix():
    """Gibbs invariance: Lie at dt = 1 has the exact equilibrium law, so the
    time-averaged coverage equals the transfer matrix (P:1046-1052 at desk scale)."""
    N, beta, K, hp = 2048, 2.0, 1.0, 1.5
    hd = exact.h_dyn_from_paper(hp, K, 1)
    sim = FSKMC(1, (N,), (32,), "adsdes", model_params(ca=1, cd=1, beta=beta, K=K, h=hd),
                colours=2, replicas=4, seed=9)
    sim.run(30.0, 1.0, "lie")
    covs = []
    for _ in range(60):
        sim.run(1.0, 1.0, "lie")
        covs.append(sim.get_config().mean())
    covs = np.array(covs)
    batch = covs.reshape(6, 10).mean(axis=1)
    se = batch.std(ddof=1) / math.sqrt(len(batch))
    target = exact.paper_cov1d(beta, K, hp)
    assert abs(covs.mean() - target) <= max(Z * se, 5e-3)


def test_o2_deterministic_and_resumable():
    """Global ids: run(T1); run(T2) == run(T1+T2) bit-exactly; same seed same result."""
    p = model_params(ca=1, cd=1, beta=1.5, K=1, h=-2)
    init = (np.random.default_rng(0).random((1, 32, 32)) < 0.5).astype(np.uint8)
    a = FSKMC(2, (32, 32), (4, 4), "adsdes", p, seed=1)
    a.set_config(init); a.run(3.0, 1.0, "strang")
    b = FSKMC(2, (32, 32), (4, 4), "adsdes", p, seed=1)
    b.set_config(init); b.run(1.0, 1.0, "strang"); b.run(2.0, 1.0, "strang")
    assert np.array_equal(a.get_config(), b.get_config())
    assert a.events == b.events and a.window == b.window == 9
    assert int(a.W_events.sum()) == a.events            # P9: sum_m W[m] = events


def test_o2_diffusion_conserves_particles():
    """P9: pure Kawasaki hops (c_a = c_d = 0) conserve particle number exactly."""
    p = model_params(ca=0.0, cd=0.0, beta=1.0, K=1.0, h=0.0, c_hop=1.0)
    init = (np.random.default_rng(2).random((2, 16, 16)) < 0.3).astype(np.uint8)
    sim = FSKMC(2, (16, 16), (4, 4), "adsdes_diff", p, replicas=2, seed=4)
    sim.set_config(init)
    sim.run(5.0, 0.5, "strang")
    assert sim.events > 0
    assert np.array_equal(sim.get_config().sum(axis=(1, 2)), init.sum(axis=(1, 2)))


@pytest.mark.parametrize("kind", list(MODELS_1D))
def test_o1_law_vs_exact_generator(kind):
    """O1 samples e^{T Q} (eq.(generator), eq.(semigroup))."""
    N, T, R = 5, 0.7, 12000
    p = MODELS_1D[kind]
    lat = bf.Lattice(1, 1, N, 1, 1, 2)
    Q, Qc, S = bf.generators(bf_model(kind, p), lat)
    start = np.array([1, 0, 0, 2 if S == 3 else 1, 0], np.uint8)
    law = bf.evolve(bf.point_mass(S, N, start), Q, T)
    idx = []
    for r in range(R):
        snap, _ = ssa_snapshots(start.reshape(1, N), 1, kind, model_params(**p), [T], seed=77, stream=r)
        idx.append(confs_index(snap, S)[0])
    check_law(np.array(idx), law)


def test_o1_noninteracting_closed_form():
    p = model_params(ca=1.0, cd=0.5, beta=1.0, K=0.0, h=0.0)
    snap, nev = ssa_snapshots(np.zeros((1, 4096), np.uint8), 1, "adsdes", p, [0.5, 1.0, 4.0], seed=3)
    for k, t in enumerate([0.5, 1.0, 4.0]):
        th = exact.noninteracting_theta(t, 1.0, 0.5)
        assert abs(snap[k].mean() - th) <= Z * math.sqrt(th * (1 - th) / 4096)


@pytest.mark.parametrize("inner", ["lie", "strang"])
def test_o2_multiscale_law(inner):
    """f2: O2's spatio-temporal scheme (eq.(strang3)) samples the brute-force law exactly."""
    N, q, dt, T, R, nf = 8, 2, 0.5, 1.0, 20000, 3
    p = dict(ca=0.4, cd=0.6, beta=1.0, K=1.0, h=-1.0, c_hop=3.0)
    lat = bf.Lattice(1, 1, N, 1, q, 2)
    m = bf_model("adsdes_diff", p)
    Qf, Qfc, S = bf.generators(m, lat, mech="fast")
    Qs, Qsc, _ = bf.generators(m, lat, mech="slow")
    start = np.array([1, 1, 0, 0, 1, 0, 0, 1], np.uint8)
    law = bf.law_multiscale(bf.point_mass(S, N, start), Qsc, Qfc, dt, T, nf, inner, 2)
    sim = FSKMC(1, (N,), (q,), "adsdes_diff", model_params(**p), colours=2, replicas=R, seed=31)
    sim.set_config(np.broadcast_to(start, (R, 1, N)))
    sim.run_multiscale(T, dt, nf, inner)
    check_law(confs_index(sim.get_config(), S), law)


@pytest.mark.parametrize("outer,inner,n_inner", [("lie", "lie", 2), ("strang", "strang", 2), ("lie", "strang", 1)])
def test_o2_nested_law(outer, inner, n_inner):
    """f3: O2's nested scheme (eq.(opdecomp2), R28) samples the brute-force law exactly
    (1D ring of 8 single-site cells, outer blocks of 2 cells)."""
    N, q, dt, T, R, B = 8, 1, 0.5, 1.0, 20000, 2
    p = dict(ca=1.0, cd=1.0, beta=1.0, K=1.0, h=-1.0)
    nl = bf.NestedLattice(1, 1, N, 1, q, 2, B)
    Q, Qc2, S = bf.generators(bf_model("adsdes", p), nl)
    start = np.array([1, 1, 0, 0, 1, 0, 0, 1], np.uint8)
    law = bf.law_nested(bf.point_mass(S, N, start), Qc2, 2, dt, T, n_inner, outer, inner)
    sim = FSKMC(1, (N,), (q,), "adsdes", model_params(**p), colours=2, replicas=R, seed=41)
    sim.set_config(np.broadcast_to(start, (R, 1, N)))
    sim.run_nested(T, dt, n_inner, outer, inner, B)
    check_law(confs_index(sim.get_config(), S), law)
    assert sim.window == 2 * (len(bf._inner(inner, 2, 1.0)) * n_inner * (2 if outer == "lie" else 3))
    assert int(sim.W_events.sum()) == sim.events


def test_o2_zgb_odiff_o_hops_conserve_oxygen():
    """P9 for the O-diffusion model (R33): windows restricted to the O-hop classes (the fast factor
    of eq.(strang3)) move O atoms onto vacant neighbours only -- the O count per replica is
    conserved exactly, no CO appears, and events do happen."""
    init = np.zeros((2, 16, 16), np.uint8)
    rng = np.random.default_rng(8)
    init[rng.random((2, 16, 16)) < 0.4] = 2
    p = model_params(k1=0.4, k2=1.0, c_hop=1.5)
    sim = FSKMC(2, (16, 16), (4, 4), "zgb_odiff", p, replicas=2, seed=12)
    sim.set_config(init)
    hop = {i for i in range(sim.table["n"]) if int(sim.table["type"][i]) == 8}
    assert len(hop) == 4 and all(sim.table["rate"][i] == 1.5 for i in hop)
    for colour in range(4):
        sim.substep(colour, 0.7, hop)
    out = sim.get_config()
    assert sim.events > 0
    assert np.array_equal((out == 2).sum(axis=(1, 2)), (init == 2).sum(axis=(1, 2)))
    assert (out == 1).sum() == 0


@pytest.mark.parametrize("inner", ["lie", "strang"])
def test_o2_multiscale_law_zgb_odiff(inner):
    """f2 on the model the paper names: ZGB with fast O diffusion, the O hops as the
    fast mechanism of eq.(strang3); O2's law = the brute-force law (8-site ring, 3^8 states)."""
    N, q, dt, T, R, nf = 8, 2, 0.5, 1.0, 20000, 3
    p = dict(k1=0.45, k2=1.0, c_hop=2.5)
    lat = bf.Lattice(1, 1, N, 1, q, 2)
    m = bf_model("zgb_odiff", p)
    Qf, Qfc, S = bf.generators(m, lat, mech="fast")
    Qs, Qsc, _ = bf.generators(m, lat, mech="slow")
    assert Qf.nnz > 0 and S == 3
    start = np.array([2, 0, 1, 2, 0, 0, 2, 0], np.uint8)
    law = bf.law_multiscale(bf.point_mass(S, N, start), Qsc, Qfc, dt, T, nf, inner, 2)
    sim = FSKMC(1, (N,), (q,), "zgb_odiff", model_params(**p), colours=2, replicas=R, seed=32)
    sim.set_config(np.broadcast_to(start, (R, 1, N)))
    sim.run_multiscale(T, dt, nf, inner)
    check_law(confs_index(sim.get_config(), S), law)
