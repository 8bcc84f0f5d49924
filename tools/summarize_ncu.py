"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py ROUND_TAG CONFIG prof_test.ncu-rep [prof_encode.ncu-rep ...]
                                  [--launches gpurun_out/launches.csv]

Writes profiles/<tag>_<kernel>.md with the key counters and the top stall
sites, and merges the trigger kernel's DRAM traffic per launch into
profiles/traffic.json (read by bench.py's roofline.traffic).
"""
from __future__ import annotations

import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("lts__t_sectors_srcunit_tex_op_read.sum", "L2 read sectors (from L1)"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput %"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1TEX throughput %"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "global load sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum", "global store sectors"),
    ("l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum", "local (spill) load sectors"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard stall / issue"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "short-scoreboard stall / issue"),
    ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "MIO-throttle stall / issue"),
    ("smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio", "math-pipe-throttle stall / issue"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
]


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra], capture_output=True, text=True)
    return list(csv.reader(io.StringIO(out.stdout)))


def summarize(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else os.path.basename(rep)
    got = {}
    for m, label in METRICS:
        if m in hdr:
            i = hdr.index(m)
            got[m] = (label, vals[i], units[i])
    sass = ncu_csv(rep, "source", ("--print-source", "sass"))
    stalls = []
    if len(sass) > 2:
        h = sass[1]
        ix = {k: i for i, k in enumerate(h)}
        data = sass[2:]
        key = "Warp Stall Sampling (All Samples)"
        tot = sum(float(r[ix[key]] or 0) for r in data)
        for r in sorted(data, key=lambda r: -float(r[ix[key]] or 0))[:12]:
            stalls.append((r[ix["Source"]].strip(), float(r[ix[key]] or 0) / max(tot, 1) * 100,
                           r[ix["Instructions Executed"]], r[ix.get("L2 Theoretical Sectors Global", 0)]))
    return name, got, stalls


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    tag, config, *reps = sys.argv[1:]
    launches = None
    if "--launches" in reps:
        i = reps.index("--launches")
        launches = reps[i + 1]
        reps = reps[:i] + reps[i + 2:]
    os.makedirs(PROF, exist_ok=True)
    traffic_path = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for rep in reps:
        name, got, stalls = summarize(rep)
        short = "k_test" if "k_test" in name else ("k_encode" if "k_encode" in name else "kernel")
        lines = [f"# {tag} {config} — `{name}`", "", f"ncu --set full --clock-control none (one launch, "
                 f"cold-cache, serialised) from `{os.path.basename(rep)}`", "", "| metric | value |", "|---|---|"]
        for m, (label, v, u) in got.items():
            lines.append(f"| {label} (`{m}`) | {v} {u} |")
        lines += ["", "Top stall sites (share of warp-stall samples):", "", "| SASS | % samples | executed | L2 sectors |",
                  "|---|---|---|---|"]
        for src, pct, ex, sec in stalls:
            lines.append(f"| `{src[:70]}` | {pct:.1f} | {ex} | {sec} |")
        with open(os.path.join(PROF, f"{tag}_{config}_{short}.md"), "w") as fh:
            fh.write("\n".join(lines) + "\n")
        if short == "k_test":
            rd = got.get("dram__bytes_read.sum")
            wr = got.get("dram__bytes_write.sum")
            if rd and wr:
                traffic[config] = to_bytes(rd[1], rd[2]) + to_bytes(wr[1], wr[2])
            sec = got.get("lts__t_sectors_srcunit_tex_op_read.sum")
            if sec:  # L2 sectors the launch read (the gather-bound roofline in bench.py)
                traffic[config + "_l2_read_sectors"] = float(sec[1])
    with open(traffic_path, "w") as fh:
        json.dump(traffic, fh, indent=1)
    if launches:
        rows = list(csv.reader(open(launches)))
        hi = None
        for i, r in enumerate(rows):
            if "Kernel Name" in r:
                hi = i
                break
        if hi is not None:
            h = rows[hi]
            kn, mv = h.index("Kernel Name"), h.index("Metric Value")
            agg = {}
            for r in rows[hi + 1:]:
                if len(r) > mv:
                    k = r[kn].split("(")[0]
                    agg.setdefault(k, []).append(float(r[mv].replace(",", "")))
            tot = sum(sum(v) for v in agg.values())
            lines = [f"# {tag} {config} launch list (ncu --metrics gpu__time_duration.sum)", "",
                     "| kernel | launches | total | share |", "|---|---|---|---|"]
            for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
                lines.append(f"| `{k}` | {len(v)} | {sum(v):.0f} | {sum(v) / tot * 100:.1f}% |")
            with open(os.path.join(PROF, f"{tag}_{config}_launches.md"), "w") as fh:
                fh.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
