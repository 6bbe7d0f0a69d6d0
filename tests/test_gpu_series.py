"""GPU tests of the f1 coverage process (kmc_record_coverage / kmc_coverage_series /
kmc_coverage_stats, reading R30).

Parity: the recorded series is bit-exact to O2's (integer counts at every macro-step boundary, the
lattice itself being bit-exact); the device statistics equal oracle/series.py's estimator on the
same series (histogram exact, mean / autocovariance within 1e-12 relative: FP64, another summation
order).  Statistics: the non-interacting closed forms (cfg1 shape, acf(l) = e^{-(ka+kd) l dt},
N C ~ Binomial(N, theta)); the 1D Ising process at small dt against the exact serial SSA (O1),
the paper's "approximations converge as dt -> 0".
"""
import numpy as np
import pytest

import synth_inputs as si
from oracle import series
from oracle.fskmc import FSKMC, model_params
from oracle.ssa import ssa_snapshots

pytestmark = pytest.mark.gpu
Z = 4.5


def _kmc():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1105_4673_b200 as kmc
    return kmc


def check_stats(g, ser, nsite, max_lag, first, bins):
    got = g.coverage_stats(max_lag, first=first, bins=bins)
    ref = series.stats(ser, nsite, max_lag, first=first, bins=bins)
    assert np.array_equal(got["hist"], ref["hist"])
    assert got["mean"] == pytest.approx(ref["mean"], rel=1e-12, abs=1e-15)
    assert got["var"] == pytest.approx(ref["var"], rel=1e-10, abs=1e-15)
    assert np.allclose(got["acf"], ref["acf"], rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("ndim,dims,cell,kind,params,scheme,dt,T,R,state", [
    (1, (512,), (16,), "adsdes", dict(ca=1.0, cd=1.0, beta=2.0, K=1.0, h=-1.5), "lie", 0.5, 5.0, 6, 1),
    (1, (256,), (4,), "zgb", dict(k1=0.4, k2=1.0), "random", 0.5, 3.0, 5, 2),
    (2, (64, 64), (8, 8), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "strang", 1.0, 4.5, 3, 0),
    (2, (32, 64), (4, 8), "zgb_diff", dict(k1=0.45, k2=1.0, c_hop=1.0), "lie", 0.25, 1.0, 2, 1),
])
def test_series_bit_exact_and_stats(ndim, dims, cell, kind, params, scheme, dt, T, R, state):
    """Sample 0 at record time, one per macro-step (a shortened last one included, T = 4.5 with
    dt = 1); counts == O2's; device statistics == the oracle estimator on the same series."""
    kmc = _kmc()
    g = kmc.KMC(ndim, dims, cell, kind=kind, replicas=R, seed=77, **params)
    o = FSKMC(ndim, dims, cell, kind, model_params(**params), replicas=R, seed=77)
    lat = (si.bernoulli_lattice(g.local_shape, 0.4, seed=3) if g.nstates == 2
           else si.categorical_lattice(g.local_shape, [0.6, 0.2, 0.2], seed=3))
    g.set_config(lat)
    o.set_config(lat)
    nmac = int(np.ceil(T / dt - 1e-9))
    g.record_coverage(nmac + 5, state=state)
    g.run(T, dt, scheme)
    ref = series.record(o, T, dt, scheme, state=state)
    got = g.coverage_series()
    assert got.shape == (nmac + 1, R)
    assert np.array_equal(got, ref)
    nsite = int(np.prod(dims))
    check_stats(g, got, nsite, min(3, nmac), 0, nsite + 1)
    check_stats(g, got, nsite, 1, 2, 7)


def test_series_capacity_restart_and_multiscale():
    """Samples beyond the capacity are dropped; re-recording restarts at the current state;
    run_multiscale and run_nested append one sample per macro-step too."""
    kmc = _kmc()
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0, c_hop=1.0)
    g = kmc.KMC(2, (32, 32), (4, 4), kind="adsdes_diff", replicas=2, seed=5, **p)
    o = FSKMC(2, (32, 32), (4, 4), "adsdes_diff", model_params(**p), replicas=2, seed=5)
    lat = si.bernoulli_lattice(g.local_shape, 0.5, seed=8)
    g.set_config(lat)
    o.set_config(lat)
    g.record_coverage(3)
    g.run(5 * 0.5, 0.5, "lie")
    o.run(5 * 0.5, 0.5, "lie")
    assert g.coverage_series().shape == (3, 2)
    g.record_coverage(10)
    g.run_multiscale(2.0, 1.0, 3, "strang")
    ref = series.record(o, 2.0, 1.0, step=lambda d: o.run_multiscale(d, d, 3, "strang"))
    assert np.array_equal(g.coverage_series(), ref)
    g.record_coverage(10, state=0)
    g.run_nested(1.0, 0.5, 2, "strang", "lie", block=2)
    ref = series.record(o, 1.0, 0.5, state=0, step=lambda d: o.run_nested(d, d, 2, "strang", "lie", block=2))
    assert np.array_equal(g.coverage_series(), ref)
    g.record_coverage(0)
    assert g.coverage_series().shape == (0, 2)


def test_series_errors():
    kmc = _kmc()
    g = kmc.KMC(1, (64,), (8,), kind="adsdes", replicas=2, K=1.0)
    with pytest.raises(kmc.KmcError):
        g.record_coverage(4, state=2)                 # adsdes has states 0, 1
    with pytest.raises(kmc.KmcError):
        g.coverage_stats(0)                           # nothing recorded
    g.record_coverage(4)
    g.run(2.0, 1.0)
    with pytest.raises(kmc.KmcError):
        g.coverage_stats(3)                           # max_lag >= n - first
    with pytest.raises(kmc.KmcError):
        g.coverage_stats(0, first=3)
    with pytest.raises(kmc.KmcError):
        g.coverage_stats(0, bins=66)                  # > N + 1
    assert g.coverage_stats(2, bins=65)["hist"].sum() == 3 * 2


def test_series_virtual_ranks_sum_to_one_rank():
    """Virtual ranks record their slab's partial counts; they sum to the G = 1 series."""
    kmc = _kmc()
    p = dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0)
    one = kmc.KMC(2, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=4, **p)
    grp = kmc.VGroup(4, (64, 32), (8, 8), kind="adsdes", replicas=2, seed=4, **p)
    lat = si.bernoulli_lattice(one.local_shape, 0.5, seed=1)
    one.set_config(lat)
    grp.set_config(lat)
    one.record_coverage(8)
    for rk in grp.ranks:
        rk.record_coverage(8)
    one.run(3.0, 1.0)
    grp.run(3.0, 1.0)
    total = sum(rk.coverage_series() for rk in grp.ranks)
    assert np.array_equal(total, one.coverage_series())
    with pytest.raises(kmc.KmcError):
        grp.ranks[0].coverage_stats(1)


def test_cfg1_noninteracting_acf_and_distribution_closed_form():
    """cfg1 shape (1D N = 1024, Q = 32, M = 1000, K = 0, c_d = 0.5), stationary Bernoulli(theta)
    start, Lie dt = 0.1: the splitting is exact for K = 0, so acf(l) = e^{-(ka+kd) l dt} (Fig.
    autocorr1D's observable) and the pooled count histogram is Binomial(N, theta) (Fig. pdf2d's)."""
    kmc = _kmc()
    N, q, M, dt, nstep = 1024, 32, 1000, 0.1, 200
    ca, cd = 1.0, 0.5
    theta = ca / (ca + cd)
    g = kmc.KMC(1, (N,), (q,), kind="adsdes", replicas=M, seed=21, ca=ca, cd=cd, beta=1.0, K=0.0, h=0.0)
    g.set_config(si.bernoulli_lattice(g.local_shape, theta, seed=6))
    g.record_coverage(nstep + 1)
    g.run(nstep * dt, dt, "lie")
    ser = g.coverage_series()
    L = 10
    st = g.coverage_stats(L, bins=N + 1)
    # SE from 10 replica batches through the oracle estimator (the device stats == oracle, above)
    parts = np.array([series.stats(b, N, L)["acf"] for b in np.array_split(ser[:, :500], 10, axis=1)])
    se = parts.std(axis=0, ddof=1) / np.sqrt(10) / np.sqrt(2)   # pooled M = 1000 vs batches of 50
    for l in range(1, L + 1):
        ex = series.noninteracting_acf(l * dt, ca, cd)
        assert abs(st["acf"][l] - ex) < Z * se[l] + 2e-3, (l, st["acf"][l], ex, se[l])
    assert st["var"] == pytest.approx(theta * (1 - theta) / N, rel=0.05)
    # histogram vs Binomial(N, theta): bins holding >= 1 % of the mass, within Z SE of the
    # expected count (samples of a replica are correlated: SE inflated by sqrt(1 + 2 sum acf))
    pmf = series.binomial_pmf(N, theta)
    nobs = st["hist"].sum()
    infl = np.sqrt(1 + 2 * sum(series.noninteracting_acf(l * dt, ca, cd) for l in range(1, 200)))
    big = pmf * nobs > 0.01 * nobs
    exp_c = pmf[big] * nobs
    assert np.all(np.abs(st["hist"][big] - exp_c) < Z * infl * np.sqrt(exp_c) + 5), "histogram vs Binomial"


def test_1d_ising_acf_vs_exact_ssa():
    """1D Ising (Fig. autocorr1D: beta = 4, h_paper = 1, R9 h_dyn = h_paper - 2K), N = 64, Q = 8: the
    coverage autocorrelation of the GPU's process at Lie dt = 0.1, sampled every 0.5 time units
    after a burn-in of 50, vs the exact SSA's (O1) at the same times, for lags 0.5 .. 8 (the acf
    decays from ~0.96 to ~0.55 there): within Z SE of the difference (replica-batch SEs)."""
    kmc = _kmc()
    N, q, dt, burn, stride, nobs = 64, 8, 0.1, 50.0, 5, 80
    prm = dict(ca=1.0, cd=1.0, beta=4.0, K=1.0, h=1.0 - 2.0)
    lags = (1, 2, 4, 8, 16)
    L = max(lags)
    M, Ms = 800, 400
    g = kmc.KMC(1, (N,), (q,), kind="adsdes", replicas=M, seed=8, **prm)
    g.set_config(si.bernoulli_lattice(g.local_shape, 0.5, seed=4))
    g.run(burn, 1.0, "lie")                                   # burn-in (coarse steps)
    g.record_coverage(nobs * stride + 1)
    g.run(nobs * stride * dt, dt, "lie")
    gpu = g.coverage_series()[::stride][: nobs + 1]
    ssa = np.zeros((nobs + 1, Ms), dtype=np.int64)
    lat0 = si.bernoulli_lattice((Ms, 1, N), 0.5, seed=12)
    times = [burn + i * stride * dt for i in range(nobs + 1)]
    for r in range(Ms):
        snaps, _ = ssa_snapshots(lat0[r], 1, "adsdes", model_params(**prm), times, seed=99, stream=r)
        ssa[:, r] = snaps.reshape(nobs + 1, -1).sum(axis=1)

    def acf_se(ser, nb):
        full = series.stats(ser, N, L)["acf"]
        parts = np.array([series.stats(b, N, L)["acf"] for b in np.array_split(ser, nb, axis=1)])
        return full, parts.std(axis=0, ddof=1) / np.sqrt(nb)

    ag, sg = acf_se(gpu, 10)
    as_, ss = acf_se(ssa, 10)
    assert as_[L] < 0.8 and ag[1] > 0.9                       # the lags span the decay
    for l in lags:
        assert abs(ag[l] - as_[l]) < Z * np.hypot(sg[l], ss[l]), (l, ag[l], as_[l], sg[l], ss[l])
