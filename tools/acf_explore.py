# exploration: coverage acf of the 1D Ising process (Fig. autocorr1D: beta = 4, h_paper = 1) at
# Lie dt = 1, 0.5, 0.1 on the GPU vs the exact SSA, sampled every 0.5 time units
import sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_1105_4673_b200 as kmc, synth_inputs as si
from oracle import series
from oracle.ssa import ssa_snapshots
from oracle.fskmc import model_params
N, q = 64, 8
prm = dict(ca=1.0, cd=1.0, beta=4.0, K=1.0, h=-1.0)
burn, dtau, nobs = 50.0, 0.5, 80
lags = [1, 2, 4, 8, 16, 32]
def acf_se(ser, nb):
    L = max(lags)
    full = series.stats(ser, N, L)["acf"]
    parts = np.array([series.stats(b, N, L)["acf"] for b in np.array_split(ser, nb, axis=1)])
    return full, parts.std(axis=0, ddof=1) / np.sqrt(nb)
res = {}
for dt in (1.0, 0.5, 0.1):
    M = 400
    g = kmc.KMC(1, (N,), (q,), kind="adsdes", replicas=M, seed=8, **prm)
    g.set_config(si.bernoulli_lattice(g.local_shape, 0.5, seed=4))
    g.run(burn, dt, "lie")
    stride = int(round(dtau / dt)) if dt < dtau else 1
    step = dt if dt >= dtau else dt
    g.record_coverage(nobs * stride + 1)
    g.run(nobs * stride * dt, dt, "lie")
    ser = g.coverage_series()[::stride][: nobs + 1] if dt < dtau else g.coverage_series()
    res[dt] = acf_se(ser, 10), (dt if dt >= dtau else dtau)
Ms = 200
ssa = np.zeros((nobs + 1, Ms), dtype=np.int64)
lat0 = si.bernoulli_lattice((Ms, 1, N), 0.5, seed=12)
times = [burn + i * dtau for i in range(nobs + 1)]
for r in range(Ms):
    snaps, _ = ssa_snapshots(lat0[r], 1, "adsdes", model_params(**prm), times, seed=99, stream=r)
    ssa[:, r] = snaps.reshape(nobs + 1, -1).sum(axis=1)
(as_, ss) = acf_se(ssa, 8)
print("mean coverage ssa", ssa.mean() / N)
for dt, ((a, s), tau) in res.items():
    for l in lags:
        li = int(round(l * dtau / tau))
        if li <= max(lags):
            print(f"dt={dt} lag_time={l * dtau:5.1f} gpu {a[li]:.4f}+-{s[li]:.4f}  ssa {as_[l]:.4f}+-{ss[l]:.4f}  diff {a[li] - as_[l]:+.4f}")
