"""Regenerate the round-2 result tables of profiles/README.md, DESIGN.md §13 and README.md from the
committed bench lines (profiles/round2_bench_*.json) and ncu per-unit figures
(profiles/substep_profile.json).  Run here after copying a bench_all run into profiles/."""
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
prof = json.load(open(os.path.join(P, "substep_profile.json")))


def line(name):
    return json.loads(open(os.path.join(P, f"round2_bench_{name}.json")).read().strip().splitlines()[-1])


def frac(d, key):
    r = d["roofline"]
    if key not in prof:
        return None
    epl = r["algorithmic"]["events_per_launch"]
    return prof[key]["warp_inst_per_event"] * epl / (r["avg_launch_ms"] / 1e3) / 1e9 / r["peak"]


ROWS = [  # (label, bench file stem, profile key, summary, launch list)
    ("ising2d_32768_strang", "ising2d_32768_strang", "ising2d_32768_strang"),
    ("ising2d_32768", "ising2d_32768", "ising2d_32768"),
    ("ising2d_32768 --dt 0.01", "ising2d_32768_dt0.01", "ising2d_32768@dt0.01"),
    ("zgb2d_32768", "zgb2d_32768", "zgb2d_32768"),
    ("zgbdiff2d_32768", "zgbdiff2d_32768", "zgbdiff2d_32768"),
    ("zgbodiff2d_32768", "zgbodiff2d_32768", "zgbodiff2d_32768"),
    ("diff2d_8192", "diff2d_8192", "diff2d_8192"),
    ("diff2d_8192 --dt 0.1", "diff2d_8192_dt0.1", "diff2d_8192@dt0.1"),
    ("ising2d_1024", "ising2d_1024", "ising2d_1024"),
]


def profiles_table():
    out = ["| Workload | bench line | events/s | site-updates/s | e2e events/s | frac | alg | hbm | warp-inst/event | ncu issue active | regs | ncu summary | launch list |",
           "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for label, stem, key in ROWS:
        d = line(stem)
        p = prof[key]
        out.append(f"| `{label}` | `round2_bench_{stem}.json` | {d['value']:.3g} | {d['site_updates_per_s']:.3g} | "
                   f"{d['e2e']['value']:.3g} | {frac(d, key):.3f} | {d['roofline']['frac_algorithmic']:.3f} | "
                   f"{d['roofline']['hbm']['frac']:.4f} | {p['warp_inst_per_event']:.2f} | {p['issue_active_pct']:.0f} % | "
                   f"{p['registers']:.0f} | `round2_substep_{key}.md` | `round2_launches_{key}.csv` |")
    return "\n".join(out)


if __name__ == "__main__":
    print(profiles_table())
    for stem in ("ising1d_65536", "ising1d_65536x64", "noninteracting1d_1024x1000"):
        d = line(stem)
        print(stem, f"{d['value']:.3g} {d['site_updates_per_s']:.3g} {d['e2e']['value']:.3g} {d['ms_per_step']:.4g}")
    d = line("ising2d_32768_strang")
    print("cpu", d["cpu_baseline"]["value"], d["cpu_baseline"]["o2_single_thread"]["value"],
          d["cpu_baseline"].get("o1_single_thread", {}).get("value"))
    r = json.loads(open(os.path.join(P, "round2_bench_reference.json")).read())
    print("reference", r["value"])
