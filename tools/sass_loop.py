"""Print the instruction count of the main event loop (largest backward branch span) of a kernel
in libkmc_b200.so, with an opcode histogram: a cheap pre-GPU check of per-event cost."""
import collections
import os
import re
import subprocess
import sys

lib = os.environ.get("KMC_B200_LIB", "paper_1105_4673_b200/libkmc_b200.so")
want = sys.argv[1] if len(sys.argv) > 1 else "ILi0ELi2ELi256ELi4ELb0ELb0ELb0E"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
for f in funcs:
    name = f.split("\n", 1)[0].strip()
    if want not in name:
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,})\*/\s+([^;]*);", f)
    addr = [(int(a, 16), t.strip()) for a, t in ins]
    best = None
    for a, t in addr:
        m = re.search(r"BRA (0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) < a:
            span = (int(m.group(1), 16), a)
            if best is None or span[1] - span[0] > best[1] - best[0]:
                best = span
    body = [t for a, t in addr if best[0] <= a <= best[1]]
    step = 0
    for t in body:                      # the event step: loop head up to the first warp vote
        step += 1
        if "VOTE" in t:
            break
    ops = collections.Counter()
    for t in body[:step]:
        t = re.sub(r"^@!?U?P\w+\s+", "", t)
        ops[t.split()[0].split(".")[0]] += 1
    print(name, "loop", hex(best[0]), hex(best[1]), len(body), "instructions; event step", step)
    print(" ".join(f"{k}:{v}" for k, v in ops.most_common()))
