#!/usr/bin/env python
"""Summaries of ncu output for profiles/ (run here, on the CPU side).

  python profiles/summarize_ncu.py rep  X.ncu-rep  "source note" > profiles/<name>.json
  python profiles/summarize_ncu.py launches launches.csv [steps] > profiles/<name>.json

`rep`: selected raw metrics of every kernel in an `ncu --set full` capture plus
the SASS opcode mix and warp-stall samples by reason (from the source page).
`launches`: per-kernel launch counts, summed durations and share of the
captured launches, from the `--metrics gpu__time_duration.sum` launch list
(cold-cache, serialised: compare shares, not absolute times).
"""
import collections
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__shared_mem_per_block_static",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__waves_per_multiprocessor",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second", "sm__cycles_active.avg",
    "smsp__inst_executed.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def _csv(args):
    out = subprocess.run(["ncu", "-i", *args, "--csv"], capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def rep(path, note):
    rows = _csv([path, "--page", "raw"])
    hdr, units = rows[0], rows[1]
    kernels = {}
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?")
        key = f"{name} grid={d.get('launch__grid_size', '?')}"
        kernels[key] = {m: [d.get(m), units[hdr.index(m)] if m in hdr else ""] for m in METRICS if m in d}
    # SASS opcode mix and stall samples (source page)
    src = _csv([path, "--page", "source", "--print-source", "sass"])
    mix, stalls = collections.Counter(), collections.Counter()
    h = None
    for r in src:
        if "Source" in r and "Instructions Executed" in r:
            h = r
            continue
        if h is None or len(r) < len(h):
            continue
        d = dict(zip(h, r))
        ins = d["Source"].strip().split()
        if not ins:
            continue
        op = ins[1] if ins[0].startswith("@") and len(ins) > 1 else ins[0]
        mix[op.split(".")[0]] += int(d["Instructions Executed"] or 0)
        for k, v in d.items():
            if k.startswith("stall_") and "Not Issued" not in k and v:
                stalls[k] += int(v)
    tot = sum(mix.values()) or 1
    return {"source": note, "kernels": kernels,
            "sass_mix_top": {k: [v, round(100.0 * v / tot, 2)] for k, v in mix.most_common(12)},
            "stall_samples": dict(stalls.most_common(12))}


def launches(path, steps=1):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            k = d["Kernel Name"].split("(")[0]
            agg.setdefault(k, []).append(float(d["Metric Value"]) / 1000.0)
    total = sum(sum(v) for v in agg.values()) or 1
    return {"source": path, "unit": "us (cold-cache, serialised)",
            "kernels": {k: {"launches": len(v), "sum_us": round(sum(v), 2), "share": round(sum(v) / total, 4),
                            "first_us": [round(x, 2) for x in v[:4]]} for k, v in agg.items()}}


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        print(json.dumps(rep(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""), indent=1))
    else:
        print(json.dumps(launches(sys.argv[2]), indent=1))
