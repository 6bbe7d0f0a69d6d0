"""Summarise an ncu capture of substep_kernel into profiles/ (run here, no GPU needed).

python tools/ncu_summary.py --rep gpurun_out/prof.ncu-rep --bench gpurun_out/plain.log \
       --tag round2 [--launches gpurun_out/launches.csv]

Writes/updates profiles/substep_profile.json ({workload[@dt]: {...}}, read by bench.py for the
roofline per-unit figure) and profiles/<tag>_substep_<workload[@dt]>.md (human-readable summary).
"""
import argparse
import csv
import io
import json
import os
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

METRICS = {
    "gpu__time_duration.sum": "duration",
    "inst_executed": "warp_inst",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "threads_per_inst",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__registers_per_thread": "registers",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}
UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1}


def read_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in METRICS:
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            d[METRICS[h]] = x * UNITS.get(u, 1)
    stalls = {}
    for h, v in zip(hdr, vals):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls[h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = float(v)
            except ValueError:
                pass
    return d, stalls


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rep", required=True)
    ap.add_argument("--bench", required=True, help="bench.py JSON log of the same command")
    ap.add_argument("--kind", default=None, help="profile key (default: the bench line's workload[@dt])")
    ap.add_argument("--tag", default="round1")
    ap.add_argument("--launches", default=None)
    a = ap.parse_args()
    d, stalls = read_raw(a.rep)
    b = json.loads(open(a.bench).read().strip().splitlines()[-1])
    if a.kind is None:
        import sys
        sys.path.insert(0, ROOT)
        import synth_inputs as si
        w = b["config"]["workload"]
        a.kind = w if b["config"]["dt"] == si.WORKLOADS[w]["dt"] else f"{w}@dt{b['config']['dt']:g}"
    C = b["config"].get("colours", 2)
    lps = {"lie": C, "strang": 2 * C - 1, "random": C}[b["config"].get("scheme", "lie")]   # windows per step
    ev_launch = b["events_per_step"] / lps
    ipe = d["warp_inst"] / ev_launch            # the captured launch against the mean launch
    ipe_src = "captured launch / mean events per launch"
    # preferred: instructions summed over the timed steps' launches (launch list with
    # smsp__inst_executed.sum) / the events of those steps -- exact for schedules whose windows
    # differ in duration (Strang half steps)
    if a.launches and os.path.exists(a.launches):
        per = {}
        for r in csv.reader(open(a.launches)):
            if len(r) > 14 and r[0].isdigit() and "substep_kernel" in r[4] and r[12] == "smsp__inst_executed.sum":
                per[int(r[0])] = float(r[14].replace(",", ""))
        if per:
            ids = sorted(per)
            warm, steps = b.get("warmup", 3), b.get("steps", 2)
            timed = ids[warm * lps:(warm + steps) * lps]
            if len(timed) == steps * lps:
                ipe = sum(per[i] for i in timed) / (b["events_per_step"] * steps)
                ipe_src = f"launch list: instructions of the {len(timed)} timed launches / their events"
    ipe_note = ipe_src
    summary = {
        "warp_inst_per_event": round(ipe, 3),
        "warp_inst_per_event_source": ipe_note,
        "thread_inst_per_event": round(ipe * d.get("threads_per_inst", 32), 1),
        "events_per_launch": ev_launch,
        "dram_bytes_per_launch": d.get("dram_read", 0) + d.get("dram_write", 0),
        "ncu_duration_ms": d["duration"] * 1e3,
        "lane_efficiency": d.get("threads_per_inst", 0) / 32.0,
        **{k: d.get(k) for k in ("issue_active_pct", "warps_active_pct", "registers", "fp64_pipe_pct",
                                 "alu_pipe_pct", "xu_pipe_pct", "dram_throughput_pct")},
        "stalls_per_issue": {k: round(v, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1]) if v > 0.02},
        "source": os.path.basename(a.rep), "workload": b["config"]["workload"],
    }
    pj = os.path.join(ROOT, "profiles", "substep_profile.json")
    allp = json.load(open(pj)) if os.path.exists(pj) else {}
    allp[a.kind] = summary
    os.makedirs(os.path.dirname(pj), exist_ok=True)
    json.dump(allp, open(pj, "w"), indent=1)
    md = [f"# {a.tag}: substep_kernel ncu summary ({a.kind}, {b['config']['workload']})", "",
          f"Command: `python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 1` under",
          "`ncu --set full --clock-control none --import-source on -k regex:substep -s 6 -c 1` (one launch).", "",
          "| quantity | value |", "|---|---|"]
    for k, v in summary.items():
        if k != "stalls_per_issue":
            md.append(f"| {k} | {v} |")
    md += ["", "Warp stall reasons (warps stalled per issued instruction):", ""]
    md += [f"- {k}: {v}" for k, v in summary["stalls_per_issue"].items()]
    if a.launches and os.path.exists(a.launches):
        rows = [r for r in csv.reader(open(a.launches)) if len(r) > 14 and r[0].isdigit()
                and r[12] == "gpu__time_duration.sum"]
        tot = {}
        for r in rows:
            name = r[4].split("(")[0].replace("void ", "")
            tot[name] = tot.get(name, 0.0) + float(r[14].replace(",", ""))
        s = sum(tot.values())
        md += ["", "Launch list (ncu gpu__time_duration.sum, cold-cache serialised; shares of the listed launches):", ""]
        md += [f"- {k}: {v / 1e6:.3f} ms total, {100 * v / s:.1f} %" for k, v in sorted(tot.items(), key=lambda x: -x[1])]
    out = os.path.join(ROOT, "profiles", f"{a.tag}_substep_{a.kind}.md")
    open(out, "w").write("\n".join(md) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
