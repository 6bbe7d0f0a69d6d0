"""Time the pieces of the e2e step (set_config from pinned host memory, run, observables)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1105_4673_b200 as kmc
import synth_inputs as si
wl = si.WORKLOADS["ising2d_32768"]
k = kmc.KMC(2, wl["dims"], wl["cell"], kind="adsdes", seed=1, stream=torch.cuda.current_stream().cuda_stream, **wl["params"])
lat = si.bernoulli_lattice(k.local_shape, 0.5)
host = torch.from_numpy(lat).pin_memory()
hn = host.numpy()
print("pinned:", host.is_pinned())
for it in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    k.set_config(hn); t1 = time.perf_counter()
    k.observables(); t2 = time.perf_counter()
    k.run(1.0, 1.0, "lie"); torch.cuda.synchronize(); t3 = time.perf_counter()
    k.observables(); t4 = time.perf_counter()
    print(f"set_config {1e3*(t1-t0):.1f} ms  obs {1e3*(t2-t1):.1f}  run {1e3*(t3-t2):.1f}  obs {1e3*(t4-t3):.1f}")
t = torch.empty(lat.size, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize(); t0 = time.perf_counter(); t.copy_(host.view(-1), non_blocking=True); torch.cuda.synchronize()
print("torch H2D 1 GiB ms", 1e3 * (time.perf_counter() - t0))
