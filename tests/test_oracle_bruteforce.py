"""Pins of the brute-force master equation and the closed forms (CPU).

The brute-force generator (oracle/bruteforce.py) is checked against what the
paper and the mathematics fix: the non-interacting two-state law, the
transfer matrix / eq.(exactcov1d), detailed balance (Gibbs invariance,
P:981-985), generator additivity (eq.(gendecomp)), Lie/Strang local orders
(eq.(error), eq.(error2)), the random-PCS mean error and the
paper's printed closed-form values (tests/golden/paper_closed_forms.txt).
"""
import math
import os

import numpy as np
import pytest
import scipy.sparse as sp
from scipy.linalg import expm

from oracle import bruteforce as bf
from oracle import exact

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def ising(beta=1.0, K=1.0, h=-1.0, ca=1.0, cd=1.0):
    return dict(kind="adsdes", ca=ca, cd=cd, beta=beta, K=K, h=h)


def test_golden_paper_closed_forms():
    rows = [l.split() for l in open(os.path.join(GOLDEN, "paper_closed_forms.txt"))
            if l.strip() and not l.startswith("#")]
    for kind, b, h, val, tol in rows:
        b, h, val, tol = float(b), float(h), float(val), float(tol)
        if kind == "cov1d":
            got = exact.paper_cov1d(b, 1.0, h)
        elif kind == "cov2d":
            got = exact.paper_cov2d(b, 1.0)
        else:
            got = exact.beta_c(1.0)
        assert abs(got - val) <= tol, (kind, b, h, got, val)


def test_generator_rows_sum_to_zero_and_additivity():
    lat = bf.Lattice(1, 1, 6, 1, 2, 2)
    Q, Qc, S = bf.generators(ising(), lat)
    assert np.abs(np.asarray(Q.sum(axis=1))).max() < 1e-12
    assert abs(Q - (Qc[0] + Qc[1])).max() < 1e-12          # eq.(gendecomp)
    assert (Qc[0] - sp.diags(Qc[0].diagonal())).min() >= 0.0


def test_noninteracting_closed_form_all_schemes():
    """K = 0: [L^E, L^O] = 0 so every scheme is exact; per-site law is the
    two-state closed form theta(t)."""
    lat = bf.Lattice(1, 1, 6, 1, 1, 2)
    m = ising(beta=1.0, K=0.0, h=0.3, ca=1.0, cd=0.5)
    Q, Qc, S = bf.generators(m, lat)
    p0 = bf.point_mass(S, lat.N, [0] * lat.N)
    cov = bf.coverage_values(lat, S)
    th = exact.noninteracting_theta(1.5, 1.0, 0.5, 1.0, 0.3)
    for scheme in ("exact", "lie", "strang"):
        p = bf.law(p0, Q, Qc, scheme, 0.5, 1.5, 2)
        assert abs(p @ cov - th) < 1e-9, scheme
    # random (SL) schedule: a site's colour is active in B ~ Binomial(C n, 1/C) of the
    # C n windows, so its law is E_B[theta(B dt)] (eq.(SLPCS))
    n, C, dt = 3, 2, 0.5
    thr = sum(math.comb(C * n, b) * (1 / C) ** b * (1 - 1 / C) ** (C * n - b)
              * exact.noninteracting_theta(b * dt, 1.0, 0.5, 1.0, 0.3) for b in range(C * n + 1))
    p = bf.law(p0, Q, Qc, "random", dt, n * dt, C)
    assert abs(p @ cov - thr) < 1e-9


def test_gibbs_invariance_and_transfer_matrix():
    """Detailed balance (R9): pi Q^c = 0 for every colour; the stationary
    coverage equals the finite-N transfer matrix of the literal rates."""
    N = 8
    lat = bf.Lattice(1, 1, N, 1, 2, 2)
    m = ising(beta=1.3, K=1.0, h=-0.4, ca=1.0, cd=0.7)
    Q, Qc, S = bf.generators(m, lat)
    A = Q.toarray()
    w, v = np.linalg.eig(A.T)
    pi = np.real(v[:, np.argmin(np.abs(w))])
    pi = pi / pi.sum()
    for Qk in Qc:
        assert np.abs(pi @ Qk.toarray()).max() < 1e-12
    cov = bf.coverage_values(lat, S)
    tm = exact.tm_coverage_1d(N, 1.3, 1.0, -0.4, 1.0, 0.7)
    assert abs(pi @ cov - tm) < 1e-12


def test_transfer_matrix_vs_paper_formula_R9():
    """Thermodynamic-limit TM of the literal rates equals eq.(exactcov1d) with the
    R9 mapping h_paper = h_dyn + 2K."""
    for beta in (1.0, 2.0, 4.0):
        for hp in (0.0, 0.5, 1.0, 1.5, 2.0):
            hd = exact.h_dyn_from_paper(hp, 1.0, 1)
            assert abs(exact.tm_coverage_1d(None, beta, 1.0, hd) - exact.paper_cov1d(beta, 1.0, hp)) < 1e-12


def _defect(Q, Qc, dt, scheme):
    E = expm(dt * Q.toarray())
    A, B = Qc[0].toarray(), Qc[1].toarray()
    if scheme == "lie":
        P = expm(dt * A) @ expm(dt * B)
    else:
        P = expm(0.5 * dt * A) @ expm(dt * B) @ expm(0.5 * dt * A)
    return np.abs(E - P).max()


def test_local_error_orders():
    """eq.(error): Lie local error O(dt^2); eq.(error2): Strang O(dt^3)."""
    lat = bf.Lattice(1, 1, 6, 1, 1, 2)
    Q, Qc, S = bf.generators(ising(beta=1.0, K=1.0, h=-1.0, ca=0.2, cd=0.2), lat)
    dt = 0.05
    rl = _defect(Q, Qc, dt, "lie") / _defect(Q, Qc, dt / 2, "lie")
    rs = _defect(Q, Qc, dt, "strang") / _defect(Q, Qc, dt / 2, "strang")
    assert 3.6 < rl < 4.4
    assert 7.2 < rs < 8.8


def test_random_pcs_mean_error():
    """E_xi[e^{dt A_xi1} e^{dt A_xi2}] - e^{dt(A1+A2)} = 1/4 (A1 - A2)^2 dt^2 + O(dt^3)."""
    lat = bf.Lattice(1, 1, 4, 1, 1, 2)
    Q, Qc, S = bf.generators(ising(beta=1.0, K=1.0, h=-1.0), lat)
    A1, A2 = Qc[0].toarray(), Qc[1].toarray()
    for dt in (1e-2, 5e-3):
        avg = 0.25 * sum(expm(dt * X) @ expm(dt * Y) for X in (A1, A2) for Y in (A1, A2))
        err = avg - expm(dt * (A1 + A2))
        pred = 0.25 * (A1 - A2) @ (A1 - A2) * dt * dt
        assert np.abs(err - pred).max() < 10 * dt ** 3 * np.abs(A1).max() ** 3


def test_boundary_only_commutator():
    """eq.(opdecomperror): [L^E, L^O] is supported on cell boundaries -- with
    K = 0 (no interaction across cells) it vanishes."""
    lat = bf.Lattice(1, 1, 6, 1, 2, 2)
    Q, Qc, S = bf.generators(ising(K=0.0, h=0.2), lat)
    A, B = Qc[0].toarray(), Qc[1].toarray()
    assert np.abs(A @ B - B @ A).max() < 1e-12
    Q, Qc, S = bf.generators(ising(K=1.0, h=-1.0), lat)
    A, B = Qc[0].toarray(), Qc[1].toarray()
    assert np.abs(A @ B - B @ A).max() > 1e-3


def test_lie_error_one_over_q_and_random_ratio_P6():
    """eq.(liebound): the Lie coverage error is O(1/q) -- on the N = 12 ring (c_a = c_d = 1,
    beta = K = 1, h = -1, empty start, T = 2, dt = 1) error x q is constant to 15 % for q = 1, 2, 3, 6
    (-0.0303, -0.0133, -0.0088, -0.0044); eq.(pcscompare): the random schedule's
    error exceeds Lie's by a factor growing with q (dt_Lie ~ q dt_Random)."""
    N = 12
    errs, ratios = [], []
    for q in (1, 2, 3, 6):
        lat = bf.Lattice(1, 1, N, 1, q, 2)
        Q, Qc, S = bf.generators(ising(beta=1.0, K=1.0, h=-1.0), lat)
        p0 = bf.point_mass(S, N, [0] * N)
        cov = bf.coverage_values(lat, S)
        ex = bf.law(p0, Q, Qc, "exact", 0, 2.0, 2) @ cov
        lie = bf.law(p0, Q, Qc, "lie", 1.0, 2.0, 2) @ cov - ex
        rnd = bf.law(p0, Q, Qc, "random", 1.0, 2.0, 2) @ cov - ex
        errs.append(lie * q)
        ratios.append(rnd / lie)
    assert abs(errs[1] - (-0.0266)) < 5e-4 and abs(errs[3] - (-0.0264)) < 5e-4
    assert max(errs) - min(errs) < 0.15 * abs(np.mean(errs))
    assert all(r2 > r1 for r1, r2 in zip(ratios, ratios[1:])) and ratios[0] > 3


def test_lie_order_asymmetric_start():
    """Global weak error of Lie is O(dt) with an asymmetric start (R#-P5), Strang O(dt^2)."""
    lat = bf.Lattice(1, 1, 8, 1, 2, 2)
    Q, Qc, S = bf.generators(ising(beta=1.0, K=1.0, h=-1.0), lat)
    conf = [1 if lat.colour(i) == 1 else 0 for i in range(lat.N)]
    p0 = bf.point_mass(S, lat.N, conf)
    cov = bf.coverage_values(lat, S)
    ex = bf.law(p0, Q, Qc, "exact", 0, 2.0, 2) @ cov
    el = [abs(bf.law(p0, Q, Qc, "lie", dt, 2.0, 2) @ cov - ex) for dt in (0.25, 0.125)]
    es = [abs(bf.law(p0, Q, Qc, "strang", dt, 2.0, 2) @ cov - ex) for dt in (0.25, 0.125)]
    assert 1.6 < el[0] / el[1] < 2.5
    assert 3.2 < es[0] / es[1] < 5.0


def test_tm_correlation_vs_bruteforce_and_paper_R15():
    """f1 pins: the finite-N transfer-matrix E[s_0 s_r] equals the brute-force stationary law of the
    literal rates (N = 8 ring), and the R15 reading of eq.(exactcorr1d) equals the N -> infinity TM."""
    N = 8
    lat = bf.Lattice(1, 1, N, 1, 2, 2)
    m = ising(beta=1.7, K=1.0, h=-0.6, ca=1.0, cd=0.9)
    Q, Qc, S = bf.generators(m, lat)
    w, v = np.linalg.eig(Q.toarray().T)
    pi = np.real(v[:, np.argmin(np.abs(w))])
    pi /= pi.sum()
    import itertools
    confs = np.array(list(itertools.product(range(2), repeat=N)))[:, ::-1]
    for r in range(0, 5):
        bfv = pi @ (confs[:, 0] * confs[:, r % N])
        assert abs(bfv - exact.tm_correlation_1d(N, 1.7, 1.0, -0.6, r, 1.0, 0.9)) < 1e-12
    for beta, hp in ((2.0, 1.0), (4.0, 1.0), (1.0, 0.3)):
        hd = exact.h_dyn_from_paper(hp, 1.0, 1)
        for r in (0, 1, 2, 5, 9):
            assert abs(exact.paper_corr1d_corrected(beta, 1.0, hp, r) - exact.tm_correlation_1d(None, beta, 1.0, hd, r)) < 1e-12


def test_oracle_correlation_counts_by_definition():
    """FSKMC.correlation counts equal a direct double loop over sites (definition)."""
    from oracle.fskmc import FSKMC, model_params
    rng = np.random.default_rng(5)
    o = FSKMC(2, (8, 12), (2, 2), "zgb", model_params(), replicas=2)
    o.set_config(rng.integers(0, 3, (2, 8, 12)).astype(np.uint8))
    for state in (0, 1, 2):
        c = o.correlation(7, state)
        for r in range(8):
            bx = sum(int(o.lat[k, y, x] == state and o.lat[k, y, (x + r) % 12] == state)
                     for k in range(2) for y in range(8) for x in range(12))
            by = sum(int(o.lat[k, y, x] == state and o.lat[k, (y + r) % 8, x] == state)
                     for k in range(2) for y in range(8) for x in range(12))
            assert c["x"][r] == bx and c["y"][r] == by


def test_multiscale_generator_split_and_order():
    """f2 (eq.(fastslow), eq.(strang3)): L = L_fast + L_slow exactly (per colour), and the
    spatio-temporal scheme with Strang inside is second order: halving dt quarters the global error."""
    lat = bf.Lattice(1, 1, 6, 1, 2, 2)
    m = dict(kind="adsdes_diff", ca=0.4, cd=0.6, beta=1.0, K=1.0, h=-1.0, c_hop=3.0)
    Q, Qc, S = bf.generators(m, lat)
    Qf, Qfc, _ = bf.generators(m, lat, mech="fast")
    Qs, Qsc, _ = bf.generators(m, lat, mech="slow")
    assert abs(Q - Qf - Qs).max() < 1e-12
    for c in range(2):
        assert abs(Qc[c] - Qfc[c] - Qsc[c]).max() < 1e-12
        assert abs(Qfc[c]).max() > 0 and abs(Qsc[c]).max() > 0
    start = [1, 1, 0, 0, 1, 0]
    p0 = bf.point_mass(S, 6, start)
    cov = bf.coverage_values(lat, S, sites=[0, 1])           # a sub-lattice observable (P5)
    ex = bf.law(p0, Q, Qc, "exact", 0, 1.0, 2) @ cov
    e = [abs(bf.law_multiscale(p0, Qsc, Qfc, dt, 1.0, 3, "strang", 2) @ cov - ex) for dt in (0.25, 0.125)]
    assert 3.0 < e[0] / e[1] < 5.5, e


def test_nested_generator_split_and_inner_order():
    """f3 (eq.(sublatt2), eq.(opdecomp2), R28): the 2C nested generators L^{o,c} sum
    to L and, over o, to each cell-colour generator L^c; as n_inner grows the nested scheme
    converges to the outer scheme with EXACT outer factors e^{D L^o}, at second order with a
    Strang inner scheme and first order with Lie (ratios 4 and -> 2 per doubling of n_inner)."""
    m = ising(beta=1.0, K=1.0, h=-1.0)
    lat = bf.Lattice(1, 1, 8, 1, 1, 2)
    nl = bf.NestedLattice(1, 1, 8, 1, 1, 2, 2)
    Q, Qc, S = bf.generators(m, lat)
    Q2, Qc2, _ = bf.generators(m, nl)
    assert len(Qc2) == 4
    assert abs(Q - Q2).max() < 1e-12
    for c in range(2):
        assert abs(Qc[c] - Qc2[c] - Qc2[2 + c]).max() < 1e-12
    # cell 0 (x = 0) is in outer block 0, cell colour 0; cell 2 in outer block 1
    assert nl.colour(0) == 0 and nl.colour(1) == 1 and nl.colour(2) == 2 and nl.colour(3) == 3
    p0 = bf.point_mass(S, 8, [1, 1, 0, 0, 1, 0, 0, 1])
    cov = bf.coverage_values(lat, S, sites=[0, 1])
    QE, QO = Qc2[0] + Qc2[1], Qc2[2] + Qc2[3]
    dt, T = 0.5, 1.0
    for outer, seq in (("lie", [(0, dt), (1, dt)]), ("strang", [(0, dt / 2), (1, dt), (0, dt / 2)])):
        p = p0.copy()
        for _ in range(2):
            for o, d in seq:
                p = bf.evolve(p, [QE, QO][o], d)
        ref = p @ cov
        es = [abs(bf.law_nested(p0, Qc2, 2, dt, T, n, outer, "strang") @ cov - ref) for n in (2, 4, 8)]
        el = [abs(bf.law_nested(p0, Qc2, 2, dt, T, n, outer, "lie") @ cov - ref) for n in (4, 8)]
        assert 3.8 < es[0] / es[1] < 4.2 and 3.8 < es[1] / es[2] < 4.2, (outer, es)
        assert 1.9 < el[0] / el[1] < 2.9, (outer, el)


def test_nested_noninteracting_exact_and_gibbs_invariance():
    """K = 0: all nested generators commute, so the nested scheme is exact (closed form theta);
    spin flip: pi L^{o,c} = 0 for each of the 2C nested generators (detailed balance, R9)."""
    nl = bf.NestedLattice(1, 1, 8, 1, 1, 2, 2)
    m0 = ising(beta=1.0, K=0.0, h=0.3, ca=1.0, cd=0.5)
    Q, Qc2, S = bf.generators(m0, nl)
    p0 = bf.point_mass(S, 8, [0] * 8)
    cov = bf.coverage_values(nl, S)
    th = exact.noninteracting_theta(1.5, 1.0, 0.5, 1.0, 0.3)
    for outer, inner, n in (("lie", "lie", 1), ("lie", "strang", 3), ("strang", "lie", 2)):
        assert abs(bf.law_nested(p0, Qc2, 2, 0.5, 1.5, n, outer, inner) @ cov - th) < 1e-9
    m = ising(beta=1.3, K=1.0, h=-0.4, ca=1.0, cd=0.7)
    Q, Qc2, S = bf.generators(m, nl)
    w, v = np.linalg.eig(Q.toarray().T)
    pi = np.real(v[:, np.argmin(np.abs(w))])
    pi = pi / pi.sum()
    for Qk in Qc2:
        assert np.abs(pi @ Qk.toarray()).max() < 1e-12


def test_workload_cdf_partition_pins():
    """f4 (R29): closed forms of the cdf re-partition.  Uniform load -> the even split;
    odd-number loads w_s = 2s+1 (cdf (s+1)^2/M^2) -> b_l = ceil(M sqrt(l/P)); each group's load is
    at most S/P + max_s w_s (the cdf mapping's defining property); the loads add up to S."""
    from oracle import workload as wk
    M, P = 64, 4
    b = wk.cdf_bounds(np.full(M, 7, dtype=np.uint64), P)
    assert list(b) == [0, 16, 32, 48, 64]
    w = np.arange(M, dtype=np.uint64) * 2 + 1
    b = wk.cdf_bounds(w, P)
    assert list(b) == [0] + [math.ceil(M * math.sqrt(l / P) - 1e-12) for l in range(1, P)] + [M]
    rng = np.random.default_rng(5)
    for trial in range(20):
        w = rng.integers(0, 50, size=96).astype(np.uint64) * (rng.random(96) < 0.7)
        w[rng.integers(0, 96)] += 500                                   # a hot strip
        S = int(w.sum())
        b = wk.cdf_bounds(w, 6)
        gl = wk.group_loads(w, b)
        assert int(gl.sum()) == S and np.all(np.diff(b) >= 1)
        assert gl.max() <= S / 6 + int(w.max())
    # granule 2: bounds even, every group >= 2 strips, still within the property up to 2 strips
    w = rng.integers(0, 100, size=128).astype(np.uint64)
    b = wk.cdf_bounds(w, 8, granule=2)
    assert np.all(b % 2 == 0) and np.all(np.diff(b) >= 2)
    assert wk.group_loads(w, b).max() <= w.sum() / 8 + 3 * int(w.max())
    # no events: the even split
    assert list(wk.cdf_bounds(np.zeros(12, dtype=np.uint64), 3)) == [0, 4, 8, 12]
