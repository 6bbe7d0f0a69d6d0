"""Static per-source-line instruction counts of a kernel's event step (nvdisasm -g of the in-tree
library's cubin): where the issued instructions of one event go, before spending GPU time."""
import collections
import os
import re
import subprocess
import sys
import tempfile

want = sys.argv[1] if len(sys.argv) > 1 else "_ZN3kmc14substep_kernelILi0ELi2ELi256ELi4ELb0ELb0ELb0EEEvNS_11SubstepArgsEjj"
cubin_name = sys.argv[2] if len(sys.argv) > 2 else "kmc_kernels.sm_100a.cubin"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(os.environ.get("KMC_B200_LIB", "paper_1105_4673_b200/libkmc_b200.so"))], cwd=d,
               capture_output=True)
txt = subprocess.run(["nvdisasm", "-g", os.path.join(d, cubin_name)], capture_output=True, text=True).stdout
line = None
rows = []
inside = False
labels, pending_labels = {}, []
for l in txt.splitlines():
    if l.lstrip().startswith(".section"):
        inside = (".text." + want) in l
        continue
    if not inside:
        continue
    m = re.search(r'## File "([^"]+)", line (\d+)', l)
    if m:
        line = (os.path.basename(m.group(1)), int(m.group(2)))
        continue
    m = re.match(r"^(\.L_x_\d+):", l.strip())
    if m:
        pending_labels.append(m.group(1))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", l)
    if m:
        a = int(m.group(1), 16)
        for lb in pending_labels:
            labels[lb] = a
        pending_labels = []
        rows.append((a, m.group(2).strip(), line))
# loop = largest backward branch; event step = loop head .. first VOTE
best = None
for a, t, _ in rows:
    m = re.search(r"BRA `\((\.L_x_\d+)\)", t)
    if m and m.group(1) in labels:
        tgt = labels[m.group(1)]
        if tgt < a and (best is None or a - tgt > best[1] - best[0]):
            best = (tgt, a)
region = sys.argv[3] if len(sys.argv) > 3 else "step"     # "step" or "refill" (rest of the loop)
step = []
seen_vote = False
for a, t, ln in rows:
    if a < best[0] or a > best[1]:
        continue
    if region == "step" or seen_vote:
        step.append((t, ln))
    if "VOTE" in t:
        if region == "step":
            break
        seen_vote = True
print(len(step), "instructions in the", region, "region")
cnt = collections.Counter(ln for _, ln in step)
src = {}
for (f, n), c in sorted(cnt.items(), key=lambda x: -x[1]):
    path = os.path.join("paper_1105_4673_b200/csrc", f)
    if f not in src and os.path.exists(path):
        src[f] = open(path).read().splitlines()
    text = src.get(f, [""] * (n + 1))[n - 1].strip()[:80] if f in src else ""
    print(f"{c:4d} {f}:{n:<4d} {text}")
