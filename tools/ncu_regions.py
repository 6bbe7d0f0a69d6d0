"""Executed warp-instructions and stall samples of a captured kernel split into regions: the main
event loop's event step (loop head .. first VOTE), the rest of the loop (park / write-back / refill)
and everything outside the loop.  python tools/ncu_regions.py gpurun_out/prof_zgb.ncu-rep"""
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iex, isamp = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), \
    hdr.index("Warp Stall Sampling (All Samples)")
ins = [(int(r[ia], 16), r[isrc].strip(), int(r[iex] or 0), int(r[isamp] or 0)) for r in rows[2:] if len(r) > iex]
best = None
for a, src, _, _ in ins:
    m = re.search(r"BRA (?:`\(\.L_x_\d+\)|)?\s*(0x[0-9a-f]+)", src)
    if m and int(m.group(1), 16) < a:
        span = (int(m.group(1), 16), a)
        if best is None or span[1] - span[0] > best[1] - best[0]:
            best = span
tot = sum(e for _, _, e, _ in ins)
samp = sum(s for _, _, _, s in ins)
loop = [x for x in ins if best and best[0] <= x[0] <= best[1]]
step_end = next((a for a, src, _, _ in loop if "VOTE" in src), best[1] if best else 0)
step = [x for x in loop if x[0] <= step_end]
rest = [x for x in loop if x[0] > step_end]
f = lambda xs, k: sum(x[k] for x in xs)
print(f"loop {hex(best[0])}..{hex(best[1])}, step ends {hex(step_end)}")
for name, xs in [("event step", step), ("park/write-back/refill", rest),
                 ("outside loop", [x for x in ins if not (best and best[0] <= x[0] <= best[1])])]:
    print(f"{name:24s} executed {f(xs, 2) / tot:6.1%}   stall samples {f(xs, 3) / max(1, samp):6.1%}")

if len(sys.argv) > 2:   # dump the park/refill region with executed counts and stall samples
    for a, src, e, s_ in rest:
        if e:
            print(f"{hex(a)[-5:]} {e:10d} {s_:6d}  {src}")
