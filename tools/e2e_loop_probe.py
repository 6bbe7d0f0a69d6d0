"""Per-step wall times of bench.py's e2e loop in two variants (ising2d_32768_strang): counters read
synchronously (kmc_observables) or asynchronously (kmc_observables_device + pinned copy)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1105_4673_b200 as kmc  # noqa: E402
import synth_inputs as si  # noqa: E402

wl = si.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "ising2d_32768_strang"]
stream = torch.cuda.Stream()
torch.cuda.set_stream(stream)
k = kmc.KMC(wl["ndim"], wl["dims"], wl["cell"], kind=wl["kind"], seed=1, stream=stream.cuda_stream, **wl["params"])
lat = si.bernoulli_lattice(k.local_shape, 0.5, seed=3)
packed = si.packed_lattice(lat, wl["ndim"], wl["cell"], 2 if wl["kind"].startswith("zgb") else 1)
hin = torch.from_numpy(packed.view(np.int64)).pin_memory().numpy().view(np.uint64).reshape(packed.shape)
hout = torch.empty(hin.size, dtype=torch.int64).pin_memory().numpy().view(np.uint64).reshape(packed.shape)
dt = wl["dt"]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cd = torch.zeros((N + 1, kmc.OBS_WORDS), dtype=torch.int64, device="cuda")
ch = torch.zeros((N + 1, kmc.OBS_WORDS), dtype=torch.int64).pin_memory()
for variant in ("sync", "async", "mapped", "none", "sync", "async", "mapped", "none"):
    k.stage_config_packed(hin)
    k.commit_config()
    k.run(dt, dt, wl["scheme"])
    k.observables()
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    k.stage_config_packed(hin)
    k.commit_config()
    up = variant not in ("noup", "none")
    down = variant not in ("nodown", "none")
    for s in range(N):
        if s + 1 < N and up:
            k.stage_config_packed(hin)
        k.run(dt, dt, wl["scheme"])
        if down:
            k.download_config_packed(hout)
        if variant == "sync":
            k.observables()
        elif variant != "async":
            k.observables_device(ch[s + 1].data_ptr())
        else:
            k.observables_device(cd[s + 1].data_ptr())
            ch[s + 1].copy_(cd[s + 1], non_blocking=True)
        if s + 1 < N and up:
            k.commit_config()
        t.append(time.perf_counter())
    k.download_wait()
    torch.cuda.synchronize()
    t.append(time.perf_counter())
    d = np.diff(np.array(t)) * 1e3
    print(variant, "total %.1f ms" % ((t[-1] - t[0]) * 1e3), "per-step host ms:", " ".join("%.1f" % x for x in d))
