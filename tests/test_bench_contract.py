"""bench.py contract checks that need no GPU: the reference arm's JSON line (the CPU oracle, O2, on
a bounded sample) and the per-workload config / L2 policy both arms report."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


@pytest.mark.parametrize("workload", ["ising2d_32768_strang", "ising1d_65536x64"])
def test_reference_arm_json_line(workload):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload",
                          workload, "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "events/s"
    assert d["config"]["workload"] == workload
    # the oracle as it stands on all host cores (the -fopenmp build of the same C source)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == os.cpu_count()
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_gpus_n_relaunches_one_process_per_rank():
    """`bench.py --gpus 2` without WORLD_SIZE re-launches itself under torchrun (one process per
    rank, 127.0.0.1 rendezvous); with the reference arm that runs on CPU: rank 0 alone prints one
    line with n_gpus = 2 and the other rank exits 0."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--impl", "reference",
                          "--workload", "ising1d_65536x64", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["config"]["workload"] == "ising1d_65536x64"


def test_config_and_l2_policy():
    import bench
    import synth_inputs as si
    for w in si.WORKLOADS:
        c = bench.arm_config(w, si.WORKLOADS[w]["dt"], 1)
        assert c["workload"] == w and c["l2"]
        flush, _ = bench.l2_policy(si.WORKLOADS[w], c["dims_per_gpu"])
        nplanes = 2 if si.WORKLOADS[w]["kind"].startswith("zgb") else 1
        nbytes = (__import__("numpy").prod(c["dims_per_gpu"]) * si.WORKLOADS[w].get("replicas_per_gpu", 1)
                  * nplanes / 8)
        assert flush == (nbytes < 2 * bench.L2_BYTES)
    # weak scaling grows the 2D lattice with the GPU count, strong scaling splits it
    assert bench.arm_config("ising2d_32768", 1.0, 8)["global_dims"] == [8 * 32768, 32768]
    assert bench.arm_config("ising2d_32768", 1.0, 8, scaling="strong")["dims_per_gpu"] == [4096, 32768]


def test_algorithmic_op_counts():
    """DESIGN.md §8 / SURVEY §8(d): clock draw 90 + 3 x classes; an event adds selection 6 and the
    update (4 one-site, 8 pair); 2D Ising ads/des has 7 classes -> 121 per event, 111 per cell-window."""
    import bench
    ops, pe, pw = bench.alg_ops("adsdes", 2, 10, 2)
    assert (pe, pw) == (121, 111) and ops == 10 * 121 + 2 * 111
    _, pe, _ = bench.alg_ops("zgb", 2, 1, 0)
    assert pe == 90 + 3 * 13 + 6 + 8
    import synth_inputs as si
    assert bench.DEFAULT_WORKLOAD in si.WORKLOADS and si.WORKLOADS[bench.DEFAULT_WORKLOAD]["scheme"] == "strang"
