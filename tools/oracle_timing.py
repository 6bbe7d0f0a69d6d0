"""CPU baselines on the host of the GPU box (SURVEY §8(d) "oracle timing"): O2 (serial
fractional-step oracle, single thread) and O1 (exact serial SSA, single thread) on samples of the
target workload.  Prints one JSON line.  Test infrastructure only (imports oracle/)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import synth_inputs as si  # noqa: E402
from oracle.fskmc import FSKMC, model_params  # noqa: E402
from oracle.ssa import ssa_snapshots  # noqa: E402

wl = si.WORKLOADS["ising2d_32768"]
out = {"host_cores": os.cpu_count()}
try:
    out["cpu_model"] = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
except Exception:
    pass
for side in (256, 512):
    o = FSKMC(2, (side, side), wl["cell"], "adsdes", model_params(**wl["params"]), seed=7)
    o.set_config(si.bernoulli_lattice((1, side, side), 0.5, seed=si.SEED_BASE + 1))
    t0 = time.perf_counter()
    o.run(2.0, 1.0, "lie")
    el = time.perf_counter() - t0
    out[f"O2_{side}"] = {"events": o.events, "seconds": round(el, 3), "events_per_s": o.events / el}
for side in (256,):
    lat = si.bernoulli_lattice((1, side, side), 0.5, seed=si.SEED_BASE + 1)[0]
    t0 = time.perf_counter()
    _, nev = ssa_snapshots(lat, 2, "adsdes", model_params(**wl["params"]), [2.0], seed=3)
    el = time.perf_counter() - t0
    out[f"O1_{side}"] = {"events": nev, "seconds": round(el, 3), "events_per_s": nev / el}
print(json.dumps(out))
