#!/usr/bin/env python
"""SURVEY §8(d) result table on one GPU: every config C1-C5 x value
distribution (shaped / random / ties) through bench.py, one JSON row each.

  python profiles/results_table.py > profiles/r02_results_table.json     (on a B200)

Columns: combos/s, (combination x input state) evaluations/s, plan-search ms
(device median / p10 / p90, e2e median), enumeration ms, ALU roofline
fraction, plan total (identical to the oracle's in the parity tests).
"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    rows = []
    for cfg in ["C1", "C2", "C3", "C4", "C5"]:
        for dist in ["shaped", "random", "ties"]:
            steps = "5" if cfg == "C4" else "20"
            cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--dist", dist,
                   "--steps", steps, "--no-minplus"]
            if not (dist == "shaped" and cfg in ("C1", "C2", "C3", "C5")):
                cmd.append("--no-cpu-baseline")            # 1-thread + all-core oracle on the shaped rows
            out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=900)
            line = [x for x in out.stdout.strip().splitlines() if x.startswith("{")]
            if not line:
                rows.append({"config": cfg, "dist": dist, "error": out.stderr[-400:]})
                continue
            d = json.loads(line[-1])
            ps = d.get("plan_search_ms", {})
            rows.append({
                "config": cfg, "dist": dist, "combos_per_step": d["config"].get("combos_per_step"),
                "combos_per_s": d["value"], "e2e_combos_per_s": d["e2e"]["value"],
                "device_ms_median": ps.get("device_median"), "device_ms_p10": ps.get("device_p10"),
                "device_ms_p90": ps.get("device_p90"), "e2e_ms_median": ps.get("e2e_median"),
                "e2e_ms_p10": ps.get("e2e_p10"), "e2e_ms_p90": ps.get("e2e_p90"),
                "e2e_cold_first_call_ms": ps.get("e2e_cold_first_call"),
                "phases_device_ms": ps.get("phases_device_median"),
                "enum_ms": ps.get("enum_ms_avg"), "alu_frac": d["roofline"]["frac"],
                "cpu_baseline": d.get("cpu_baseline"),
                "dtype": d["dtype"], "plan_total_ns": d.get("plan_total_ns"), "clocks": d.get("clocks"),
            })
    print(json.dumps({"source": "python profiles/results_table.py (bench.py per config x dist, 1 GPU)",
                      "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
