"""Rewrite the numeric columns of the round-2 result tables in DESIGN.md §13, README.md and
profiles/README.md from the committed bench lines and ncu figures (tools/tables.py); notes columns
and prose are left as they are."""
import json
import os
import re
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import tables as T  # noqa: E402

ROOT = T.ROOT
DESIGN_ROWS = {
    "`ising2d_32768_strang` (bench default), Strang Δt = 1": ("ising2d_32768_strang", "ising2d_32768_strang"),
    "`ising2d_32768`, Lie Δt = 1": ("ising2d_32768", "ising2d_32768"),
    "same, Δt = 0.01": ("ising2d_32768_dt0.01", "ising2d_32768@dt0.01"),
    "`zgb2d_32768`, Lie Δt = 0.1": ("zgb2d_32768", "zgb2d_32768"),
    "`zgbdiff2d_32768` (cfg5: + CO hops)": ("zgbdiff2d_32768", "zgbdiff2d_32768"),
    "`zgbodiff2d_32768` (+ fast O hops, R33)": ("zgbodiff2d_32768", "zgbodiff2d_32768"),
    "`diff2d_8192`, Strang Δt = 1": ("diff2d_8192", "diff2d_8192"),
    "`diff2d_8192 --dt 0.1` (cfg4 at Δt = 0.1)": ("diff2d_8192_dt0.1", "diff2d_8192@dt0.1"),
    "`ising2d_1024` (cfg3)": ("ising2d_1024", "ising2d_1024"),
    "`ising1d_65536` (cfg2, 1 replica)": ("ising1d_65536", None),
    "`ising1d_65536x64`": ("ising1d_65536x64", None),
    "`noninteracting1d_1024x1000` (cfg1)": ("noninteracting1d_1024x1000", None),
}
README_ROWS = {
    "`ising2d_32768_strang` (default, Strang Δt = 1)": ("ising2d_32768_strang", "ising2d_32768_strang"),
    "`ising2d_32768` (Lie Δt = 1)": ("ising2d_32768", "ising2d_32768"),
    "`ising2d_32768 --dt 0.01`": ("ising2d_32768_dt0.01", "ising2d_32768@dt0.01"),
    "`zgb2d_32768` (ZGB, Lie Δt = 0.1)": ("zgb2d_32768", "zgb2d_32768"),
    "`zgbodiff2d_32768` (ZGB + fast O diffusion)": ("zgbodiff2d_32768", "zgbodiff2d_32768"),
    "`diff2d_8192` (ads/des + diffusion, Strang)": ("diff2d_8192", "diff2d_8192"),
    "`ising2d_1024` (lane-group kernel)": ("ising2d_1024", "ising2d_1024"),
    "`ising1d_65536x64` (cfg2, 64 replicas)": ("ising1d_65536x64", None),
}


def design():
    p = os.path.join(ROOT, "DESIGN.md")
    out = []
    for ln in open(p).read().split("\n"):
        cells = ln.split(" | ")
        key = cells[0][2:] if ln.startswith("| ") else None
        if key in DESIGN_ROWS and len(cells) == 7:
            stem, pk = DESIGN_ROWS[key]
            d = T.line(stem)
            fr = (f"{T.frac(d, pk):.3f} / {d['roofline']['frac_algorithmic']:.3f} / {d['roofline']['hbm']['frac']:.3f}"
                  if pk else "—")
            cells[1:6] = [f"{d['value']:.3g}", f"{d['site_updates_per_s']:.3g}", f"{d['ms_per_step']:.3g} ms",
                          f"{d['e2e']['value']:.3g}", fr]
            ln = " | ".join(cells)
        out.append(ln)
    open(p, "w").write("\n".join(out))


def readme():
    p = os.path.join(ROOT, "README.md")
    out = []
    for ln in open(p).read().split("\n"):
        for lab, (stem, pk) in README_ROWS.items():
            if ln.startswith("| " + lab + " |"):
                d = T.line(stem)
                fr = f"{T.frac(d, pk):.2f}" if pk else "—"
                ln = f"| {lab} | {d['value']:.3g} | {d['site_updates_per_s']:.3g} | {d['e2e']['value']:.3g} | {fr} |"
        out.append(ln)
    open(p, "w").write("\n".join(out))


def profiles_readme():
    p = os.path.join(ROOT, "profiles", "README.md")
    lines = open(p).read().split("\n")
    i0 = next(i for i, l in enumerate(lines) if l.startswith("| Workload | bench line"))
    i1 = i0
    while lines[i1].startswith("|"):
        i1 += 1
    lines[i0:i1] = T.profiles_table().split("\n")
    open(p, "w").write("\n".join(lines))


if __name__ == "__main__":
    design()
    readme()
    profiles_readme()
