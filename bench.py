"""Benchmark of the fractional-step KMC hot path (BASELINE.json metric: KMC events/s).

python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--workload NAME] [--dt DT]

A step = one macro-step of the named workload's scheme (every window of every colour: SURVEY §8(a)
rows a2-a7) + the observables (a8), inputs resident in HBM.  Default workload: BASELINE's target
lattice (2D Ising ads/des 32768^2, 8x8 cells) with the Strang splitting at dt = 1 -- the paper's dt
at which the scheme also meets the north star's accuracy bar (|dtheta| <= 1e-2 vs the exact SSA,
tests/test_gpu_statistics.py; the Lie number is `--workload ising2d_32768`).  N > 1: one process per
GPU (this script re-launches itself under torchrun when WORLD_SIZE is unset), 2D slab decomposition
with the NCCL halo exchange, weak scaling (one workload-sized slab per GPU), max over ranks.
Prints ONE JSON line on rank 0.
"""
import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth_inputs as si  # noqa: E402

METRIC = "KMC events/sec (and site-updates/sec) at 1/2/4/8 B200; % of HBM peak"
UNIT = "events/s"
DEFAULT_WORKLOAD = "ising2d_32768_strang"

# Algorithmic work per unit ("Algorithmic work"): scalar operations the
# method needs, independent of this implementation.
#   one clock draw = Philox4x32-10 (10 rounds x (2 widening multiplies + 4 XOR) = 60) + U, -ln U and
#                    tau = E / lambda with the accept test (30)                              -> 90
#   lambda and the class walk over NC classes (count x rate, add, compare)                  -> 3 NC
#   an executed event adds the member selection (6) and the update (4 one-site, 8 pair events)
#   every cell-window ends with one more (rejected) clock draw (R5), which also needs lambda
ALG_CLOCK, ALG_SELECT = 90, 6
NCLASS_2D = {"adsdes": 7, "adsdes_diff": 22, "zgb": 13, "zgb_diff": 17, "zgb_odiff": 17}
NCLASS_1D = {"adsdes": 5, "adsdes_diff": 9, "zgb": 7, "zgb_diff": 9, "zgb_odiff": 9}


def alg_ops(kind, ndim, events, cell_windows):
    nc = (NCLASS_2D if ndim == 2 else NCLASS_1D)[kind]
    apply = 4 if kind == "adsdes" else 8
    per_event = ALG_CLOCK + 3 * nc + ALG_SELECT + apply
    per_window = ALG_CLOCK + 3 * nc
    return events * per_event + cell_windows * per_window, per_event, per_window


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p)), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------------------------
# CPU oracle legs (cpu_baseline and --impl reference): the O2 oracle as it stands -- the same C
# source, single-threaded (the test build) or with the cells of a colour on all host cores (built with
# -fopenmp, bit-identical results).  Only these legs execute oracle/.
# ---------------------------------------------------------------------------------------------
def cpu_model():
    try:
        return [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except Exception:
        return None


def oracle_sample(wl, sites, seed=7):
    """A bounded sample of the workload for the O2 oracle: a side x side periodic sub-lattice in 2D,
    in 1D the workload's ring (truncated to `sites`) with as many replicas as fill `sites`."""
    from oracle.fskmc import FSKMC, model_params
    if wl["ndim"] == 2:
        side = int(round(sites ** 0.5))
        side -= side % (2 * max(wl["cell"]))
        dims, R, desc = (side, side), 1, f"{side}x{side} periodic sub-lattice"
        shape = (1, side, side)
    else:
        N = min(wl["dims"][0], sites)
        R = max(1, sites // N)
        dims, desc = (N,), f"{R} x {N}-site rings"
        shape = (R, 1, N)
    o = FSKMC(wl["ndim"], dims, wl["cell"], wl["kind"], model_params(**wl["params"]), replicas=R, seed=seed)
    o.set_config(initial_lattice(wl, shape, si.SEED_BASE + 1))
    return o, desc


def initial_lattice(wl, shape, seed):
    if wl["kind"].startswith("zgb"):
        p = [1.0 - wl["init"], wl["init"] / 2, wl["init"] / 2] if wl["init"] else [1.0, 0.0, 0.0]
        return si.categorical_lattice(shape, p, seed=seed)
    return si.bernoulli_lattice(shape, wl["init"], seed=seed)


def oracle_child():
    """Child process (env BENCH_ORACLE_CHILD = JSON job): times O2 with the library ORC_LIB (the
    OpenMP build) on a sample; prints one JSON line."""
    job = json.loads(os.environ["BENCH_ORACLE_CHILD"])
    wl = si.WORKLOADS[job["workload"]]
    o, desc = oracle_sample(wl, job["sites"])
    dt = job["dt"]
    for _ in range(job.get("warmup", 0)):
        o.run(dt, dt, wl["scheme"])
    e0, t0 = o.events, time.perf_counter()
    steps, per_step = 0, []
    while steps < job["max_steps"]:
        ts = time.perf_counter()
        o.run(dt, dt, wl["scheme"])
        o.observables()
        per_step.append(time.perf_counter() - ts)
        steps += 1
        if job.get("seconds") and time.perf_counter() - t0 >= job["seconds"]:
            break
    el = time.perf_counter() - t0
    print(json.dumps({"events": o.events - e0, "seconds": el, "steps": steps, "desc": desc,
                      "threads": int(os.environ.get("OMP_NUM_THREADS", "1"))}), flush=True)


def run_oracle_child(job, threads):
    """O2 in a child process: threads > 1 -> the -fopenmp build of the same source on `threads` cores."""
    env = dict(os.environ, BENCH_ORACLE_CHILD=json.dumps(job), OMP_NUM_THREADS=str(threads))
    if threads > 1:
        from oracle import _build as ob
        env["ORC_LIB"] = ob.build_openmp(os.path.join(ROOT, "oracle", "_fskmc_oracle_omp.so"))
    else:
        env.pop("ORC_LIB", None)
    r = subprocess.run([sys.executable, os.path.abspath(__file__)], env=env, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle child failed: {r.stderr[-400:]}")
    return json.loads(r.stdout.strip().splitlines()[-1])


def cpu_baseline_sample(wl_name, dt):
    """cpu_baseline: O2 x all host cores on a bounded sample (~12 s), plus O2 x 1 and O1 x 1 (~5 s each)."""
    wl = si.WORKLOADS[wl_name]
    cores = os.cpu_count() or 1
    side_cores = 1024 if wl["ndim"] == 2 else 1 << 20
    par = run_oracle_child({"workload": wl_name, "dt": dt, "sites": side_cores ** 2 if wl["ndim"] == 2 else side_cores,
                            "max_steps": 1000, "seconds": 12.0}, cores)
    one = run_oracle_child({"workload": wl_name, "dt": dt, "sites": 256 * 256, "max_steps": 1000, "seconds": 5.0}, 1)
    out = {"value": par["events"] / par["seconds"], "unit": UNIT, "cores": par["threads"], "kind": "oracle",
           "sample": (f"O2 oracle (the plain C linear-scan oracle built with -fopenmp over the cells of a colour; "
                      f"bit-identical to the single-thread build) on a {par['desc']} of {wl_name}, "
                      f"{par['steps']} {wl['scheme']} macro-steps dt={dt}: {par['events']} events in "
                      f"{par['seconds']:.1f} s on {par['threads']} threads"),
           "cpu_model": cpu_model(), "host_cores": cores,
           "o2_single_thread": {"value": one["events"] / one["seconds"], "unit": UNIT, "cores": 1,
                                "sample": f"{one['desc']}, {one['steps']} macro-steps, {one['events']} events"}}
    if wl["ndim"] == 2 and wl["kind"] == "adsdes":
        from oracle.fskmc import model_params
        from oracle.ssa import ssa_snapshots
        lat = initial_lattice(wl, (1, 256, 256), si.SEED_BASE + 1)[0]
        t0 = time.perf_counter()
        _, nev = ssa_snapshots(lat, 2, wl["kind"], model_params(**wl["params"]), [40.0], seed=3)
        el = time.perf_counter() - t0
        out["o1_single_thread"] = {"value": nev / el, "unit": UNIT, "cores": 1,
                                   "sample": f"O1 exact SSA (Fenwick tree), 256x256, T = 40: {nev} events in {el:.1f} s"}
    return out


L2_BYTES = 126e6                                      # B200 L2


def l2_policy(wl, dims_per_gpu):
    """(flush?, description): a bit-packed lattice below twice the L2 is flushed out of L2 between
    timed steps (a 256 MiB buffer is written outside the per-step timing events)."""
    nplanes = 2 if wl["kind"].startswith("zgb") else 1
    nbytes = int(np.prod(dims_per_gpu)) * wl.get("replicas_per_gpu", 1) * nplanes / 8
    if nbytes >= 2 * L2_BYTES:
        return False, f"inputs larger than L2 (bit-packed lattice {nbytes / 2**20:.0f} MiB/GPU > 2 x 126 MB L2)"
    return True, (f"L2 flushed between timed steps (256 MiB written outside the per-step events; "
                  f"bit-packed lattice {nbytes / 2**20:.3g} MiB/GPU)")


def arm_config(workload, dt, world, fused=False, scaling="weak", loopback=False):
    """The `config` object of both arms (the workload the metric is quoted on)."""
    wl = si.WORKLOADS[workload]
    C = 2 if (wl["ndim"] == 1 or wl["kind"] == "adsdes") else 4
    dims = list(wl["dims"])
    if scaling == "strong" and wl["ndim"] == 2:
        per_gpu, global_dims = [dims[0] // world, dims[1]], dims
    else:
        per_gpu, global_dims = dims, ([dims[0] * world, dims[1]] if wl["ndim"] == 2 else dims)
    return {"workload": workload, "dims_per_gpu": per_gpu, "global_dims": global_dims, "cell": list(wl["cell"]),
            "model": wl["kind"], "params": wl["params"], "scheme": wl["scheme"], "dt": dt,
            "init": f"Bernoulli({wl['init']})", "colours": C,
            "replicas_per_gpu": wl.get("replicas_per_gpu", 1),
            "l2": l2_policy(wl, per_gpu)[1],
            "parallelism": (f"slab{world}" if wl["ndim"] == 2 else f"replicas{world}"),
            "exchange": ((("fused (peer writes in the window kernel)" if fused else "nccl send/recv")
                         + (" to itself (one-rank ring, NCCL loopback)" if loopback and world == 1 else ""))
                        if wl["ndim"] == 2 and (world > 1 or loopback) else "none")}


def run_reference(args):
    """--impl reference: the CPU oracle O2, timed on this host's cores, a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    wl = si.WORKLOADS[args.workload]
    dt = args.dt if args.dt is not None else wl["dt"]
    cores = os.cpu_count() or 1
    sites = 512 * 512 if wl["ndim"] == 2 else 1 << 18
    r = run_oracle_child({"workload": args.workload, "dt": dt, "sites": sites, "max_steps": args.steps,
                          "warmup": args.warmup}, cores)
    v = r["events"] / r["seconds"]
    sample = (f"O2 oracle built with -fopenmp on {r['threads']} host threads ({cpu_model()}), {r['desc']} of "
              f"{args.workload}, one {wl['scheme']} macro-step dt={dt} + observables per step")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
        "steps": r["steps"], "warmup": args.warmup, "ms_per_step": r["seconds"] * 1e3 / max(1, r["steps"]),
        "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u64+f64",
        "data": "synthetic",
        "config": arm_config(args.workload, dt, args.gpus, False, args.scaling),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": r["threads"], "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kmc", choices=["kmc", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=sorted(si.WORKLOADS))
    ap.add_argument("--dt", type=float, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="steps of the end-to-end measurement (default: --steps, raised to span >= 0.25 s of "
                         "device time so host jitter cannot dominate short steps)")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: one workload-sized slab per GPU (default); strong: the workload split over the GPUs")
    ap.add_argument("--fused-exchange", action="store_true",
                    help="N > 1: halo exchange folded into the window kernel (CUDA IPC + device flags)")
    ap.add_argument("--loopback", action="store_true",
                    help="N = 1, 2D: run the lattice as a one-rank ring through the multi-GPU data plane "
                         "(NCCL send/recv to itself, or the fused exchange) to measure its cost on one GPU")
    args = ap.parse_args()
    args.e2e_auto = args.e2e_steps is None
    if args.e2e_auto:
        args.e2e_steps = args.steps
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch this command under torchrun (the driver's own N > 1 launch
        # sets WORLD_SIZE and lands below directly); NCCL's INIT lines show the communicator size
        import random
        env = dict(os.environ)
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(random.randint(20000, 40000)),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd, env=env))
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist
    import paper_1105_4673_b200 as kmc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    uid = None
    if world == 1 and args.loopback:
        uid = kmc.nccl_unique_id()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        box = [kmc.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = box[0]

    wl = dict(si.WORKLOADS[args.workload])
    dt = args.dt if args.dt is not None else wl["dt"]
    ndim = wl["ndim"]
    strong = args.scaling == "strong"
    if ndim == 2:
        H1, W = wl["dims"]
        # weak scaling: one H1 x W slab per GPU; strong: the H1 x W lattice split over the GPUs
        gdims = (H1, W) if strong else (H1 * world, W)
    else:
        gdims = wl["dims"]
    # a dedicated stream shared with the library (kmc_dist.stream): the timing events, the device
    # observables buffer and every window are ordered on it (the legacy default stream would make
    # the library create its own stream)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    k = kmc.KMC(ndim, gdims, wl["cell"], kind=wl["kind"], replicas=wl.get("replicas_per_gpu", 1) * (world if ndim == 1 else 1),
                seed=0xB200, rank=rank, world=world, device=local, stream=stream.cuda_stream, nccl_id=uid,
                fused_exchange=args.fused_exchange and (world > 1 or args.loopback), **wl["params"])
    shape = k.local_shape
    lat = initial_lattice(wl, shape, si.SEED_BASE + rank)
    host = torch.from_numpy(lat).pin_memory()
    dev = host.to(f"cuda:{local}")
    # e2e input: the same lattice in the library's bit-packed upload format (1 bit per site and
    # plane; kmc_set_config_packed), pinned.  Conversion is input preparation, outside all timing.
    nplanes = 2 if wl["kind"].startswith("zgb") else 1
    packed = si.packed_lattice(lat, ndim, wl["cell"], nplanes)
    host_pk = torch.from_numpy(packed.view(np.int64)).pin_memory()
    host_pk_np = host_pk.numpy().view(np.uint64).reshape(packed.shape)
    # e2e result: each step's evolved packed lattice, downloaded into pinned memory
    host_out = torch.empty(host_pk.numel(), dtype=torch.int64).pin_memory()
    host_out_np = host_out.numpy().view(np.uint64).reshape(packed.shape)
    del lat, packed
    k.set_config_device(dev.data_ptr(), dev.numel())
    sites = int(np.prod(gdims)) * k.local_shape[0] * (world if ndim == 1 else 1)
    C = 2 if (ndim == 1 or wl["kind"] == "adsdes") else 4

    # a step's observables (a8) go to a device buffer (kmc_observables_device): no host round trip
    # inside the timed region; the host decodes the last snapshot afterwards
    obs_dev = torch.zeros((args.steps + 1, kmc.OBS_WORDS), dtype=torch.int64, device=f"cuda:{local}")

    def step(i):
        k.run(dt, dt, wl["scheme"])
        k.observables_device(obs_dev[i].data_ptr())

    for _ in range(max(3, args.warmup)):
        step(args.steps)
    obs0 = k.observables()
    k.enable_timing(True)
    k.timing(reset=True)
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.6)                                   # let nvidia-smi attach before the timed region
    flush, _ = l2_policy(wl, arm_config(args.workload, dt, world, args.fused_exchange, args.scaling)["dims_per_gpu"])
    if flush:
        # per-step device timing with the L2 flushed between steps, outside the events
        flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush_buf.fill_(i & 0xFF)
            evs[i][0].record(stream)
            step(i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        ms = sum(a_.elapsed_time(b_) for a_, b_ in evs)
    else:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(args.steps):
            step(i)
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    kern_ms, launches = k.timing(reset=True)
    k.enable_timing(False)
    if world > 1:
        t = torch.tensor([ms], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    obs = k.obs_decode(obs_dev[args.steps - 1].cpu().numpy())
    events = obs["events"] - obs0["events"]          # all ranks (NCCL all-reduce inside the observables)
    value = events / (ms / 1e3)
    site_updates = sites * args.steps / (ms / 1e3)

    # ---- e2e: through the public API with HOST buffers, H2D + D2H inside the timed region ----
    # Every step uploads its packed input from pinned host memory (staged on the copy stream while
    # the previous step runs, kmc_stage_config_packed / kmc_commit_config) and downloads its result:
    # the observables counters (kmc_observables_device + an asynchronous copy into pinned host memory,
    # decoded by kmc_obs_decode after the loop: no host synchronisation per step) and the evolved
    # packed lattice (kmc_download_config_packed: on its own stream, overlapping the next step, which
    # runs on the next committed configuration).  Every copy is complete inside the timed region.
    # The uploaded input is the lattice the timed steps reached (downloaded once, untimed), so every
    # e2e step runs the steady-state workload.
    if args.e2e_auto and args.e2e_steps > 0:
        # short steps (launch-bound 1D lattices, small dt): enough steps for >= 0.25 s of device time
        # (ms is the max over ranks, so every rank takes the same count)
        args.e2e_steps = max(args.e2e_steps, min(20000, math.ceil(250.0 / max(ms / args.steps, 1e-3))))
    host_pk_np[...] = k.get_config_packed()
    k.stage_config_packed(host_pk_np)                   # untimed e2e warm-up (first calls allocate
    k.commit_config()                                   # the spare planes and the copy stream)
    k.run(dt, dt, wl["scheme"])
    k.download_config_packed(host_out_np)
    k.observables()
    k.download_wait()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ne = max(1, args.e2e_steps)
    cnt_host = torch.zeros((ne + 1, kmc.OBS_WORDS), dtype=torch.int64).pin_memory()

    def counters(i):
        # the counters are written into pinned host memory by a kernel (no copy-engine transfer that
        # would queue behind the lattice download; NCCL ranks all-reduce on the device first)
        k.observables_device(cnt_host[i].data_ptr())

    t0 = time.perf_counter()
    k.stage_config_packed(host_pk_np)
    k.commit_config()
    counters(0)
    for s_ in range(args.e2e_steps):
        if s_ + 1 < args.e2e_steps:
            k.stage_config_packed(host_pk_np)          # H2D of the next step's input (pinned, packed)
        k.run(dt, dt, wl["scheme"])
        k.download_config_packed(host_out_np)          # D2H of the step's evolved lattice (async)
        counters(s_ + 1)                                # the step's counters to the host (async)
        if s_ + 1 < args.e2e_steps:
            k.commit_config()
    k.download_wait()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    cnt_np = cnt_host.numpy()
    ev_e2e = k.obs_decode(cnt_np[args.e2e_steps])["events"] - k.obs_decode(cnt_np[0])["events"]
    if world > 1:
        t = torch.tensor([e2e_s], device=f"cuda:{local}", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (substep_kernel, > 98 % of a step) ----
    peaks, peak_src = load_peaks()
    avg_launch_ms = kern_ms / max(1, launches)
    launch_s = avg_launch_ms / 1e3
    events_per_launch = events / max(1, launches) / max(1, world)      # this rank's share
    local_sites = int(np.prod(shape))
    q = wl["cell"][0] * (wl["cell"][1] if ndim == 2 else 1)
    cell_windows_per_launch = local_sites / q / C
    # (1) issue: measured warp-instructions per event (ncu launch list of this workload at this dt,
    #     profiles/substep_profile.json) x events per launch / launch time, against 148 SMs x 4
    #     schedulers x f_SM -- what the kernel executes
    prof = {}
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "substep_profile.json")))
    except Exception:
        pass
    pkey = args.workload if dt == si.WORKLOADS[args.workload]["dt"] else f"{args.workload}@dt{dt:g}"
    pent = prof.get(pkey, {})
    ipe = pent.get("warp_inst_per_event")
    sm_clk = clocks.get("sm_mhz") or peaks.get("sm_max_mhz", 1965.0)
    issue_peak = 148 * 4 * sm_clk * 1e6 / 1e9                              # G warp-inst / s
    achieved = ipe * events_per_launch / launch_s / 1e9 if ipe else None
    # (2) algorithmic: the method's scalar operations (module constants above) / 32
    #     lanes -- what an ideal lane-per-cell kernel would have to issue
    ops, ops_event, ops_window = alg_ops(wl["kind"], ndim, events_per_launch, cell_windows_per_launch)
    alg_achieved = ops / 32 / launch_s / 1e9
    # (3) HBM: SURVEY §8(d)'s algorithmic bytes (bit-packed: read the active cells + their halo, write
    #     the cells, + their halo for pair events; 1 bit per site and plane) beside the kernel's own
    #     footprint (5 words read + 1 written per active cell and plane, 8 B counter RMW)
    halo = 2 * (1 / wl["cell"][0] + 1 / wl["cell"][1]) if ndim == 2 else 2 / wl["cell"][0]
    active_sites = local_sites / C
    alg_bytes = nplanes * active_sites * ((1 + halo) + (1 if wl["kind"] == "adsdes" else 1 + halo)) / 8
    foot_bytes = cell_windows_per_launch * (nplanes * 8 * (2 * ndim + 2) + 8)
    hbm_gbs = alg_bytes / launch_s / 1e9
    roof = {"bound": "alu", "unit": "Gwarp-inst/s", "achieved": achieved, "peak": issue_peak,
            "frac": (achieved / issue_peak) if achieved else None,
            "peak_source": f"148 SMs x 4 schedulers x 1 warp-inst/clk x {sm_clk:.0f} MHz (median SM clock under load)",
            "per_unit": (f"{ipe} warp-inst/event (ncu smsp__inst_executed of this workload's launches / their events, "
                         f"profiles/substep_profile.json[{pkey}])") if ipe else f"no ncu capture for {pkey}",
            "traffic": pent.get("dram_bytes_per_launch") if ipe else None,
            "frac_algorithmic": alg_achieved / issue_peak,
            "algorithmic": {"achieved": alg_achieved, "unit": "Gwarp-inst/s",
                            "ops_per_event": ops_event, "ops_per_cell_window": ops_window,
                            "ops_per_launch": ops, "events_per_launch": events_per_launch,
                            "cell_windows_per_launch": cell_windows_per_launch,
                            "definition": "SURVEY 8(d) scalar ops (DESIGN.md 8): clock draw 90 + 3 x classes; an executed "
                                          "event + 6 selection + 4/8 update; one rejected draw ends each cell-window; / 32 lanes"},
            "ncu_pipes": ({"alu_pipe_pct": pent.get("alu_pipe_pct"), "xu_pipe_pct": pent.get("xu_pipe_pct"),
                           "fp64_pipe_pct": pent.get("fp64_pipe_pct"), "issue_active_pct": pent.get("issue_active_pct")}
                          if ipe else None),
            "kernel": "substep_kernel", "avg_launch_ms": avg_launch_ms, "launches": launches,
            "kernel_share_of_step": kern_ms / ms,
            "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": peaks["hbm_gbs"], "frac": hbm_gbs / peaks["hbm_gbs"],
                    "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": alg_bytes,
                    "algorithmic_bytes_per_site_macro_step": alg_bytes * launches / max(1, args.steps) / local_sites,
                    "kernel_footprint_bytes_per_launch": foot_bytes,
                    "dram_bytes_per_launch_ncu": pent.get("dram_bytes_per_launch") if ipe else None}}
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline_sample(args.workload, dt)
    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": max(3, args.warmup), "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "u64+f64",
        "data": "synthetic",
        "config": arm_config(args.workload, dt, world, args.fused_exchange, args.scaling, args.loopback),
        "site_updates_per_s": site_updates,
        "events_per_step": events / args.steps,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": {"value": ev_e2e / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": int(host_pk.numel() * 8),
                "d2h_bytes_per_step": int(host_out.numel() * 8) + int(cnt_host.shape[1]) * 8,
                "steps": args.e2e_steps,
                "input": "bit-packed lattice from a pinned host buffer every step (validated); the next step's upload is staged on a copy stream while the current step runs (kmc_stage_config_packed / kmc_commit_config)",
                "output": "every step's evolved bit-packed lattice to pinned host memory (kmc_download_config_packed on its own stream, overlapping the next step) + the step's observables counters (kmc_observables_device, copied asynchronously to pinned memory, decoded with kmc_obs_decode)"},
        "gpu_launches": int(launches + args.steps),
        "clocks": clocks,
    }
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    if os.environ.get("BENCH_ORACLE_CHILD"):
        oracle_child()
    else:
        main()
