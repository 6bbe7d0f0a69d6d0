"""CPU baselines on the host of the GPU box (SURVEY §8(d) "oracle timing"): O2 (serial
fractional-step oracle, single thread) and O1 (exact serial SSA, single thread) on samples of the
target workload.  Prints one JSON line.  Test infrastructure only (imports oracle/)."""
import hashlib
import json
import os
import subprocess
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
def time_o2(side, tag):
    o = FSKMC(2, (side, side), wl["cell"], "adsdes", model_params(**wl["params"]), seed=7)
    o.set_config(si.bernoulli_lattice((1, side, side), 0.5, seed=si.SEED_BASE + 1))
    t0 = time.perf_counter()
    o.run(2.0, 1.0, "lie")
    el = time.perf_counter() - t0
    out[f"{tag}_{side}"] = {"events": o.events, "seconds": round(el, 3), "events_per_s": o.events / el,
                            "lattice_sha1": hashlib.sha1(o.get_config().tobytes()).hexdigest()}


if os.environ.get("ORC_LIB"):            # child: the OpenMP build (O2 x cores)
    for side in (512, 1024):
        time_o2(side, "O2xcores")
    out["threads"] = int(os.environ.get("OMP_NUM_THREADS", "0")) or os.cpu_count()
    print(json.dumps(out))
    sys.exit(0)
for side in (256, 512):
    time_o2(side, "O2")
for side in (256,):
    lat = si.bernoulli_lattice((1, side, side), 0.5, seed=si.SEED_BASE + 1)[0]
    t0 = time.perf_counter()
    _, nev = ssa_snapshots(lat, 2, "adsdes", model_params(**wl["params"]), [2.0], seed=3)
    el = time.perf_counter() - t0
    out[f"O1_{side}"] = {"events": nev, "seconds": round(el, 3), "events_per_s": nev / el}
# O2 with the cells of a colour on all host cores (the same source built with -fopenmp; results
# identical -- the lattice hash at 512^2 must equal the single-thread run's)
from oracle import _build as ob  # noqa: E402
omp = ob.build_openmp("/tmp/_fskmc_oracle_omp.so")
env = dict(os.environ, ORC_LIB=omp, OMP_NUM_THREADS=str(os.cpu_count()))
child = subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, capture_output=True, text=True)
try:
    par = json.loads(child.stdout.strip().splitlines()[-1])
    for k, v in par.items():
        if k.startswith("O2xcores"):
            out[k] = v
    out["O2xcores_threads"] = par.get("threads")
    out["O2xcores_identical_512"] = par["O2xcores_512"]["lattice_sha1"] == out["O2_512"]["lattice_sha1"]
except Exception as e:  # noqa: BLE001
    out["O2xcores_error"] = f"{e}: {child.stderr[-300:]}"
print(json.dumps(out))
