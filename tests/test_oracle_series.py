"""Pins of the f1 coverage-process oracle (oracle/series.py, reading R30) -- CPU.

* the estimator on series whose statistics are known by hand (exact values);
* O2's recorded non-interacting process vs the closed forms (exact for the splitting: K = 0 gives
  [L^E, L^O] = 0): acf(l) = e^{-(ka+kd) l dt}, mean theta, variance theta (1 - theta) / N;
* O2's recorded interacting process (1D Ising ring, Lie) vs the brute-force autocorrelation of
  the scheme's own macro-step chain P = e^{dt Q^0} e^{dt Q^1} at stationarity.
Statistical comparisons use Z = 4.5 standard errors from replica batches.
"""
import math

import numpy as np
import pytest
from scipy.linalg import expm

import synth_inputs as si
from oracle import bruteforce as bf
from oracle import series
from oracle.fskmc import FSKMC, model_params

Z = 4.5


def test_estimator_alternating_series():
    """Coverage alternating 0, 1, 0, ... in every replica: mean 1/2, gamma(l) = (-1)^l / 4."""
    N, n, M = 5, 12, 3
    ser = np.array([[N * (i % 2)] * M for i in range(n)], dtype=np.int64)
    s = series.stats(ser, N, 6)
    assert s["mean"] == 0.5 and s["var"] == 0.25
    assert np.array_equal(s["acf"], np.array([(-1.0) ** l for l in range(7)]))


def test_estimator_constant_paths():
    """Paths constant in time, replicas at 0 and 1: every lag is fully correlated (acf = 1)."""
    N, n = 4, 9
    ser = np.array([[0, N, 0, N]] * n, dtype=np.int64)
    s = series.stats(ser, N, n - 1)
    assert s["mean"] == 0.5 and s["var"] == 0.25
    assert np.array_equal(s["acf"], np.ones(n))


def test_estimator_hand_values_and_hist():
    """counts 0, 2, 4 of N = 4: deviations -1/2, 0, 1/2 -> gamma = (1/6, 0, -1/4), acf = (1, 0, -3/2);
    histogram bins by floor(count bins / (N + 1))."""
    s = series.stats(np.array([[0], [2], [4]]), 4, 2, bins=5)
    assert s["mean"] == 0.5
    assert s["var"] == pytest.approx(1.0 / 6.0, abs=1e-15)
    assert np.allclose(s["acf"], [1.0, 0.0, -1.5], atol=1e-15)
    assert s["hist"].tolist() == [1, 0, 1, 0, 1]
    h = series.stats(np.array([[0, 1], [1, 4], [3, 4]]), 4, 0, bins=2)["hist"]
    assert h.tolist() == [3, 3]                      # 0,1,1 -> bin 0; 3,4,4 -> bin 1
    h = series.stats(np.array([[0, 1], [1, 4], [3, 4]]), 4, 1, first=1, bins=5)["hist"]
    assert h.tolist() == [0, 1, 0, 1, 2]             # samples 1..2 only


def test_estimator_errors():
    ser = np.zeros((4, 2), dtype=np.int64)
    with pytest.raises(ValueError):
        series.stats(ser, 8, 4)                       # max_lag >= n - first
    with pytest.raises(ValueError):
        series.stats(ser, 8, 0, first=4)


def batch_acf(ser, N, L, first, nb=10):
    """acf from the pooled replicas and its SE from nb replica batches."""
    full = series.stats(ser, N, L, first)["acf"]
    parts = np.array([series.stats(b, N, L, first)["acf"] for b in np.array_split(ser, nb, axis=1)])
    return full, parts.std(axis=0, ddof=1) / np.sqrt(nb)


def test_o2_noninteracting_coverage_process_closed_form():
    """K = 0, 1D, stationary Bernoulli(theta) start: the splitting is exact, so the sampled process
    has acf(l) = e^{-(ka+kd) l dt}, mean theta and variance theta (1 - theta) / N; with bins = N + 1
    the histogram is the count distribution (sum_b b hist_b = the total count)."""
    N, q, M, dt, nstep = 64, 8, 300, 0.25, 60
    ca, cd = 1.0, 0.5
    theta = ca / (ca + cd)
    o = FSKMC(1, (N,), (q,), "adsdes", model_params(ca=ca, cd=cd, beta=1.0, K=0.0, h=0.0), replicas=M, seed=11)
    o.set_config(si.bernoulli_lattice((M, 1, N), theta, seed=5))
    ser = series.record(o, nstep * dt, dt, "lie")
    assert ser.shape == (nstep + 1, M)
    s = series.stats(ser, N, 4, bins=N + 1)
    nobs = (nstep + 1) * M
    assert int((np.arange(N + 1) * s["hist"]).sum()) == int(ser.sum()) and s["hist"].sum() == nobs
    # mean: per-replica time averages are independent; their spread gives the SE
    per = ser.mean(axis=0) / N
    assert abs(s["mean"] - theta) < Z * per.std(ddof=1) / np.sqrt(M)
    assert s["var"] == pytest.approx(theta * (1 - theta) / N, rel=0.1)
    acf, se = batch_acf(ser, N, 4, 0)
    for l in range(1, 5):
        assert abs(acf[l] - series.noninteracting_acf(l * dt, ca, cd)) < Z * se[l], (l, acf[l], se[l])


def test_o2_interacting_acf_vs_bruteforce_chain():
    """1D Ising ring N = 8, cells of 2, Lie dt = 0.5: the coverage autocorrelation of O2's recorded
    process equals that of the exact macro-step chain P = e^{dt Q^0} e^{dt Q^1} started from its own
    stationary law pi (pi P = pi): (pi (f . P^l f) - (pi f)^2) / (pi f^2 - (pi f)^2)."""
    N, q, dt, M, nstep, first = 8, 2, 0.5, 2000, 30, 6
    prm = dict(ca=1.0, cd=1.0, beta=1.0, K=1.0, h=-1.0)
    lat = bf.Lattice(1, 1, N, 1, q, 2)
    Q, Qc, S = bf.generators(dict(kind="adsdes", c_hop=0.0, k1=0.4, k2=1.0, **prm), lat)
    P = expm(dt * Qc[0].toarray()) @ expm(dt * Qc[1].toarray())
    w, v = np.linalg.eig(P.T)
    pi = np.real(v[:, np.argmin(np.abs(w - 1.0))])
    pi /= pi.sum()
    f = bf.coverage_values(lat, S)
    m = pi @ f
    var = pi @ (f * f) - m * m
    Pl = np.eye(len(f))
    exact = []
    for _ in range(4):
        exact.append((pi @ (f * (Pl @ f)) - m * m) / var)
        Pl = Pl @ P
    o = FSKMC(1, (N,), (q,), "adsdes", model_params(**prm), replicas=M, seed=3)
    o.set_config(si.bernoulli_lattice((M, 1, N), 0.5, seed=9))
    ser = series.record(o, nstep * dt, dt, "lie")
    acf, se = batch_acf(ser, N, 3, first)
    assert abs(series.stats(ser, N, 0, first)["mean"] - m) < 0.02
    for l in range(1, 4):
        assert abs(acf[l] - exact[l]) < Z * se[l], (l, acf[l], exact[l], se[l])
    # the exact chain is not the K = 0 exponential: the pin sees the interaction
    assert abs(exact[1] - np.exp(-2.0 * dt)) > 0.05


def test_binomial_pmf_is_a_law():
    p = series.binomial_pmf(30, 0.3)
    assert p.sum() == pytest.approx(1.0, abs=1e-12)
    assert (np.arange(31) * p).sum() == pytest.approx(9.0, abs=1e-10)


def test_init_random_law_and_special_cases():
    """R32 initial configurations: frequencies within Z SE of p (3 states, 20k sites); p = (1, 0)
    gives the empty lattice and p = (0, 1) the full one exactly; the state of a site depends on its
    global coordinates only (a slab of rows / replicas equals the slice of the whole lattice)."""
    from oracle.init import init_random, thresholds
    p = (0.5, 0.3, 0.2)
    lat = init_random(5, 40, 100, p, seed=0x5EED)
    for s, ps in enumerate(p):
        f = (lat == s).mean()
        assert abs(f - ps) < Z * math.sqrt(ps * (1 - ps) / lat.size), (s, f)
    assert not init_random(1, 4, 8, (1.0, 0.0), seed=3).any()
    assert init_random(1, 4, 8, (0.0, 1.0), seed=3).all()
    assert thresholds((0.25, 0.75)) == [1 << 30] and thresholds((1.0, 0.0)) == [1 << 32]
    whole = init_random(3, 8, 16, (0.4, 0.6), seed=11)
    part = init_random(2, 3, 16, (0.4, 0.6), seed=11, row_offset=4, rep_offset=1)
    assert np.array_equal(part, whole[1:3, 4:7])
    with pytest.raises(ValueError):
        thresholds((0.7, 0.6, 0.1))
