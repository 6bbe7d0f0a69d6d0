"""Build the library to a scratch path (default abtmp/libkmc_b200.so) with the in-tree build's
flags, leaving the in-tree .so untouched (e.g. while a gpurun call snapshots the repo)."""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1105_4673_b200 import _build as b  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "abtmp/libkmc_b200.so"
os.makedirs(os.path.dirname(out) or ".", exist_ok=True)
cmd = ["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
       "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-shared", "-I", b.INCLUDE, "-I", b.nccl_include(),
       "-Xptxas", "-O3", "-o", out] + b.sources() + ["-ldl"] + os.environ.get("KMC_NVCC_FLAGS", "").split()
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    sys.stderr.write(r.stdout + r.stderr)
    sys.exit(1)
print(out)
