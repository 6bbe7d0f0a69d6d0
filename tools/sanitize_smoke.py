"""Small invocations of every kernel family (a quick all-paths check; also the input for
compute-sanitizer where it is available):
window kernels of all models (1D / 2D, nested, virtual ranks with the fused exchange), observables
(host and device), correlation, coverage series and statistics, random init, workload partition,
pipelined upload."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1105_4673_b200 as kmc  # noqa: E402
import synth_inputs as si  # noqa: E402

cases = [
    (2, (64, 64), (8, 8), "adsdes", dict(ca=1, cd=1, beta=1.5, K=1.0, h=-2.0), "lie"),
    (2, (32, 32), (4, 4), "adsdes_diff", dict(ca=1, cd=1, beta=1.0, K=1.0, h=-2.0, c_hop=1.0), "strang"),
    (2, (32, 32), (4, 4), "zgb", dict(k1=0.4, k2=1.0), "random"),
    (2, (32, 32), (4, 4), "zgb_diff", dict(k1=0.4, k2=1.0, c_hop=1.0), "lie"),
    (1, (512,), (16,), "adsdes", dict(ca=1, cd=1, beta=2.0, K=1.0, h=-1.0), "strang"),
]
for ndim, dims, cell, kind, p, scheme in cases:
    g = kmc.KMC(ndim, dims, cell, kind=kind, replicas=2, seed=1, **p)
    g.init_random([0.5, 0.5] if g.nstates == 2 else [0.5, 0.3, 0.2], seed=3)
    g.record_coverage(8)
    g.run(2.0, 0.5, scheme)
    buf = torch.zeros(kmc.OBS_WORDS, dtype=torch.int64, device="cuda")
    g.observables_device(buf.data_ptr())
    g.obs_decode(buf.cpu().numpy())
    g.observables(per_cell=True)
    g.correlation(4)
    g.coverage_stats(2, bins=5)
    if ndim == 2:
        g.run_nested(1.0, 0.5, 2, "lie", "lie", block=2)
    g.workload_mark()
    g.run(1.0, 0.5, scheme)
    g.workload_partition(2, 2 if ndim == 2 else 1)
    w = g.get_config_packed()
    g.stage_config_packed(w)
    g.run(0.5, 0.5, scheme)
    g.commit_config()
    g.run(0.5, 0.5, scheme)
    print(kind, ndim, "ok", flush=True)
grp = kmc.VGroup(2, (64, 32), (8, 8), kind="adsdes_diff", replicas=2, seed=2,
                 ca=1, cd=1, beta=1.0, K=1.0, h=-2.0, c_hop=1.0)
grp.set_config(si.bernoulli_lattice((2, 64, 32), 0.5, seed=1))
grp.set_fused(True)
grp.run(2.0, 0.5, "strang")
grp.observables()
print("vgroup fused ok")
torch.cuda.synchronize()
print("sanitize smoke done")
