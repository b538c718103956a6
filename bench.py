#!/usr/bin/env python
"""Benchmark: CFP plan search (combination enumeration + min-plus chain +
backtrack) on B200 -- BASELINE.json metric "strategy combos evaluated/sec and
plan-search ms (LLaMA-7B graph) at 1/2/4/8 B200".

One step = one full search of the LLaMA-7B-shaped problem (config C3,
SURVEY §8(d)): every distinct segment type's strategy combinations evaluated,
the cross terms folded, the least-index argmins, the segment chain and the
plan backtrack.  value = combos (sum over distinct types of prod_j feasible
D_j) / device time per step, inputs resident in HBM.  e2e = the same metric
through cfp_search_plan with host buffers (H2D + D2H inside).

  python bench.py [--gpus N --steps K --warmup W] [--config C3] [--impl reference]

Multi-GPU: launched under torchrun; the enumeration is sharded by prefix
range and merged by an NCCL min-allreduce inside libcfp (scaling = strong:
the problem is fixed as N grows).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from typing import Tuple

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "strategy combos evaluated/sec and plan-search ms (LLaMA-7B graph) at 1/2/4/8 B200"
UNIT = "combos/s"
# ALU-pipe roofline: VIADDMNMX.U32 issues on the ALU pipe
# at 16 lanes/clk per SM sub-partition (B300_MICROARCH.md "alu-pipe rt_SMSP=2")
# -> 4 x 16 = 64 lane-ops/clk/SM x 148 SMs x 1.965 GHz (MEASURED_PEAKS sm_max_mhz).
# The N5 microbench measured 63.8 lane-ops/clk/SM on this pool's B200.
# The layer types' loop runs on two pipes (DESIGN.md §5 "Two pipes"): of every
# three combinations one is a VIADDMNMX and two are FMA-pipe IMAD adds folded
# in by one VIMNMX3 -- its ceiling is the N5 op-3 rate measured in the same
# run (~70.6 add+mins/clk/SM; pipe rates alone would allow 96), which the
# roofline takes as the peak when it exceeds the ALU-only figure.
ALU_LANES_PER_CLK_PER_SM = 64
SMS = 148


def alu_peak_gops(sm_mhz: float) -> float:
    return ALU_LANES_PER_CLK_PER_SM * SMS * sm_mhz * 1e6 / 1e9


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """NVML sampling (every 2 ms) of SM clock and throttle reasons while the
    timed region runs (B200_PROFILING.md clocks line)."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()

    def __enter__(self):
        try:
            import pynvml as N
            N.nvmlInit()
            self.N = N
            self.h = N.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(N.nvmlDeviceGetMaxClockInfo(self.h, N.NVML_CLOCK_SM))
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        except Exception as e:  # no NVML: report nothing rather than guess
            self.N = None
            self.err = str(e)
        return self

    def _run(self):
        N = self.N
        while not self._stop.is_set():
            try:
                self.samples.append(float(N.nvmlDeviceGetClockInfo(self.h, N.NVML_CLOCK_SM)))
                try:
                    r = N.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                except AttributeError:
                    r = N.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                self.reasons |= int(r)
            except Exception:
                pass
            time.sleep(0.002)

    def __exit__(self, *a):
        self._stop.set()
        if self.N is not None:
            self.t.join(timeout=1)

    def summary(self):
        reasons = sorted(v for k, v in self.REASONS.items() if self.reasons & k)
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- helpers
def problem_bytes(prob) -> int:
    n = 0
    for t in prob.types:
        n += t.radix.nbytes + t.comp_ns.nbytes + (0 if t.comm_ns is None else t.comm_ns.nbytes)
        for e in t.edges:
            n += e.table.nbytes + 8
    for tr in prob.transitions:
        for x in tr.in_edges:
            n += x.table.nbytes + 4
    return n + prob.instances.nbytes


def plan_bytes(prob) -> int:
    N = len(prob.instances)
    kmax = max(int(len(t.radix)) for t in prob.types)
    return 8 + N * 16 + N * kmax * 4 + 4


def ncu_traffic(name, kernel):
    """DRAM bytes (read + write) of one launch of `kernel` from a committed
    `ncu --set full` summary (profiles/<name>.json, profiles/summarize_ncu.py);
    None when absent."""
    try:
        with open(os.path.join(ROOT, "profiles", name + ".json")) as fh:
            ks = json.load(fh)["kernels"]
    except Exception:
        return None
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for k, v in ks.items():
        if kernel in k:
            tot = 0.0
            for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                val, unit = v.get(m, ["0", "byte"])
                tot += float(val) * units.get(unit, 1)
            return tot
    return None


def perturbed(prob):
    """A copy of `prob` with the same structure (shapes, INF pattern, per-block
    maxima) and different values: every finite compute entry that is not its
    block's maximum and is > 0 is lowered by 1 ns."""
    import copy

    import numpy as np
    q = copy.deepcopy(prob)
    for t in q.types:
        o = t.offsets()
        for j in range(len(t.radix)):
            c = t.comp_ns[o[j]:o[j + 1]]
            m = t.comm_ns[o[j]:o[j + 1]] if t.comm_ns is not None else np.zeros_like(c)
            fin = (c != 0xFFFFFFFF) & (m != 0xFFFFFFFF)
            if not fin.any():
                continue
            w = c.astype(np.int64) + m.astype(np.int64)
            sel = fin & (w < w[fin].max()) & (c > 0)
            c[sel] -= 1
    q.name = getattr(prob, "name", "") + "+perturbed"
    return q


def combos_of(prob) -> float:
    return float(sum(prob.feasible_combinations(t) for t in prob.used_types()))


def _oracle_step_sample(prob, frac, m, cores):
    """Run the oracle over the first `frac` of every used transition's
    combination space (all input states): `frac` of a full step's oracle work."""
    from oracle import oracle as O
    used = sorted(set(int(x) for x in prob.instances))
    t0 = time.perf_counter()
    for tr in used:
        S = prob.num_combinations(prob.transitions[tr].type)
        n = max(1, min(S, int(round(S * frac))))
        O.segment_table_range(prob, tr, 0, n, nthreads=cores, m=m)
    return time.perf_counter() - t0


def _calibrate(prob, budget_s, m, cores):
    frac = 1e-7
    while True:
        dt = _oracle_step_sample(prob, frac, m, cores)
        if dt > budget_s / 8 or frac >= 1.0:
            break
        frac = min(1.0, frac * max(2.0, (budget_s / 8) / max(dt, 1e-4)))
    return min(1.0, frac * budget_s / 2 / max(dt, 1e-4))


def cpu_baseline(prob, budget_s: float = 12.0):
    """The oracle (as it stands) timed on this host's cores: a bounded sample
    (the same fraction of every used transition's combination space, all input
    states) scaled to the metric's unit."""
    from oracle import oracle as O
    O.build()
    cores = len(os.sched_getaffinity(0))
    m = O.Marshalled(prob)
    frac = _calibrate(prob, budget_s, m, cores)
    dt = _oracle_step_sample(prob, frac, m, cores)
    combos = combos_of(prob)
    # the same oracle on one thread, a smaller sample
    f1 = _calibrate(prob, budget_s / 2, m, 1)
    dt1 = _oracle_step_sample(prob, f1, m, 1)
    return {"value": combos * frac / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"first {frac:.3g} of every used transition's combination space (all input "
                      f"states), {dt:.2f} s; value = combos/step x fraction / time",
            "one_thread": {"value": combos * f1 / dt1, "unit": UNIT, "cores": 1,
                           "sample": f"first {f1:.3g} of the same spaces, {dt1:.2f} s"}}


def cpu_baseline_mem(prob, quantum, budget_s: float = 12.0):
    """The memory-constrained oracle (as it stands) on a bounded sample: the
    first fraction of every used transition's combination space (all input
    states, memory-bucketed tables), scaled to combos/s."""
    from oracle import oracle as O
    O.build()
    cores = len(os.sched_getaffinity(0))
    m = O.Marshalled(prob)
    used = sorted(set(int(x) for x in prob.instances))

    def sample(frac):
        t0 = time.perf_counter()
        for tr in used:
            S = prob.num_combinations(prob.transitions[tr].type)
            O.segment_table_mem_range(prob, tr, quantum, 0, max(1, min(S, int(round(S * frac)))),
                                      nthreads=cores, m=m)
        return time.perf_counter() - t0

    frac = 1e-7
    while True:
        dt = sample(frac)
        if dt > budget_s / 8 or frac >= 1.0:
            break
        frac = min(1.0, frac * max(2.0, (budget_s / 8) / max(dt, 1e-4)))
    frac = min(1.0, frac * budget_s / 2 / max(dt, 1e-4))
    dt = sample(frac)
    return {"value": combos_of(prob) * frac / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"memory-bucketed tables over the first {frac:.3g} of every used transition's "
                      f"combination space (all input states), {dt:.2f} s; value = combos/step x fraction / time"}


def mem_slack(prob, plan, quantum, limit):
    """Reporting only (host arithmetic on the returned plan): the plan's exact
    memory, its per-plan quanta (what the search constrains) and the
    quanta a per-block ceiling would have charged for the same plan."""
    exact = per_block = 0
    for n, t in enumerate(prob.instances):
        ty = prob.types[prob.transitions[int(t)].type]
        for j in range(len(ty.radix)):
            m = int(ty.mem_of(j)[int(plan.digits[n][j])])
            exact += m
            per_block += -(-m // quantum)
    return {"exact_kib": exact, "limit_kib": limit, "quantum_kib": quantum, "qmax": limit // quantum,
            "per_plan_quanta": int(plan.total_q), "per_plan_slack_quanta": int(plan.total_q) - exact / quantum,
            "per_block_quanta_same_plan": per_block, "per_block_slack_quanta": per_block - exact / quantum}


def flush_l2(torch, buf):
    buf.zero_()


# ---------------------------------------------------------------- arms
def workload_name(args) -> str:
    """The default arm's workload string (the reference arm reports the same)."""
    if args.config == "C3":
        return (f"{args.config}: LLaMA-7B-shaped graph, 2x4 target mesh, 34 segment instances, "
                f"4 distinct types ({args.dist} tables, seed {args.seed})")
    return f"{args.config} ({args.dist}, seed {args.seed})"


def run_reference(args, prob, rank, world):
    if rank != 0:
        return None
    from oracle import oracle as O
    O.build()
    cores = len(os.sched_getaffinity(0))
    m = O.Marshalled(prob)
    # each step: the same bounded sample, sized so that the whole run stays short
    frac = _calibrate(prob, 150.0 / max(1, args.steps + args.warmup), m, cores)
    for _ in range(args.warmup):
        _oracle_step_sample(prob, frac, m, cores)
    times = [_oracle_step_sample(prob, frac, m, cores) for _ in range(args.steps)]
    tot = sum(times)
    combos = combos_of(prob)
    value = combos * frac * args.steps / tot
    sample = (f"per step: first {frac:.3g} of every used transition's combination space "
              f"(all input states); value = combos/step x fraction / time")
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": tot / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": workload_name(args),
                       "combos_per_step": combos, "l2": "n/a (CPU oracle)"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def run_cfp(args, prob, rank, world, local_rank):
    import numpy as np
    import torch

    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    torch.cuda.set_device(local_rank)
    dist = None
    uid = None
    if world > 1:
        import torch.distributed as dist
        obj = [cfp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    ctx = cfp.Context(device=local_rank, world=world, rank=rank, nccl_unique_id=uid)
    prep = ctx.prepare(prob)
    prep.time_kernels(True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    combos = combos_of(prob)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        prep.execute()
        prep.kernel_ms()
    plan0 = prep.fetch()
    step_ms, enum_ms = [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush_l2(torch, flush)                 # L2 flushed between timed steps
            torch.cuda.synchronize()
            barrier()
            prep.execute()
            e, t = prep.kernel_ms()                # CUDA events on the library's stream
            step_ms.append(t)
            enum_ms.append(e)
        torch.cuda.synchronize()
        barrier()
    plan = prep.fetch()
    assert plan.total_ns == plan0.total_ns and np.array_equal(plan.seg_index, plan0.seg_index)
    info = prep.info()
    tot_ms = sum(step_ms)
    if dist is not None:
        t = torch.tensor([tot_ms, sum(enum_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_ms, enum_tot = float(t[0]), float(t[1])
    else:
        enum_tot = sum(enum_ms)
    clocks = clk.summary()
    # per-phase device ms (a0..a4): separate pass with an event
    # after every phase (kept out of the timed steps above)
    prep.time_kernels(2)
    phases = []
    for _ in range(max(5, min(args.steps, 10))):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        barrier()
        prep.execute()
        phases.append(prep.phase_ms())
    phase_med = {k: statistics.median(p[k] for p in phases) for k in phases[0]}
    # e2e through cfp_search_plan (host buffers in, plan out).  The calls
    # alternate between the problem and a copy with different values (same
    # structure): every call uploads its tables and recomputes everything on
    # the device; only the host-side schedule / allocation of the structure
    # is reused ("warm").  "cold" = a fresh ctx's first call (prepare incl.).
    probs = [prob, perturbed(prob)]
    want = [plan0.total_ns, None]
    e2e_ms = []
    for i in range(args.warmup + max(6, min(args.steps, 20))):
        barrier()
        t0 = time.perf_counter()
        p2 = ctx.search_plan(probs[i % 2])
        dt = (time.perf_counter() - t0) * 1e3
        if want[i % 2] is None:
            want[i % 2] = p2.total_ns
        assert p2.total_ns == want[i % 2], (i, p2.total_ns, want[i % 2])
        if i >= args.warmup:
            e2e_ms.append(dt)
    cold_ms = []
    for _ in range(3):
        c2 = cfp.Context(device=local_rank, world=world, rank=rank, nccl_unique_id=uid) if world == 1 else ctx
        barrier()
        t0 = time.perf_counter()
        p3 = c2.search_plan(probs[len(cold_ms) % 2] if world == 1 else prob)
        cold_ms.append((time.perf_counter() - t0) * 1e3)
        if c2 is not ctx:
            c2.close()
        if world > 1:
            break
    assert p3.total_ns in want
    e2e_ms.sort()
    e2e_stats = [statistics.median(e2e_ms), e2e_ms[len(e2e_ms) // 10], e2e_ms[min(len(e2e_ms) - 1, len(e2e_ms) * 9 // 10)],
                 statistics.median(cold_ms)]
    if dist is not None:
        t = torch.tensor(e2e_stats, dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_stats = [float(x) for x in t]
    e2e_med = e2e_stats[0]
    ms_per_step = tot_ms / args.steps
    value = combos / (ms_per_step * 1e-3)
    # roofline: enumeration kernels (dominant), 1 fused add+min per combination (local share)
    enum_avg_ms = enum_tot / args.steps
    achieved_gops = info.combos_local / (enum_avg_ms * 1e-3) / 1e9
    peak_alu = alu_peak_gops(1965.0)
    # N5 microbenchmarks: measured VIADDMNMX.U32 lane-op rate (ALU pipe) and
    # the two-pipe group's add+min rate on this GPU
    ip_ops, ip_ms = ctx.intpipe_bench(0, 4000)
    ip3_ops, _ = ctx.intpipe_bench(3, 4000)
    peak = max(peak_alu, ip3_ops / 1e9)
    traffic = ncu_traffic("r02_ncu_enum_v9", "enum_kernel<unsigned int, 24")
    # N2 (min,+) product microbenchmark (S in {256 .. 8192},
    # u32 / u64, with and without the least-k argmin), part of every default
    # run on rank 0 (~2 s); --no-minplus skips it
    minplus = None
    if not args.no_minplus and rank == 0:
        minplus = []
        for S in (256, 1024, 4096, 8192):
            for wide in (False, True):
                for argk in (False, True):
                    if argk and S > 4096:
                        continue
                    ms, ops = ctx.minplus_bench(S, wide=wide, iters=3 if S < 8192 else 1, argk=argk)
                    minplus.append({"S": S, "dtype": "u64" if wide else "u32", "argk": argk, "ms": ms,
                                    "addmin_per_s": ops, "frac_of_alu_peak": ops / (peak_alu * 1e9)})
    out = None
    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "u64" if info.wide_types else "u32", "data": "synthetic",
            "config": {"workload": workload_name(args),
                       "combos_per_step": combos, "l2": "flushed (512 MiB write) between timed steps",
                       "parallelism": f"enumeration sharded over {world} GPU(s), NCCL min-allreduce merge"},
            "plan_search_ms": {"device_median": statistics.median(step_ms),
                               "device_p10": sorted(step_ms)[max(0, len(step_ms) // 10)],
                               "device_p90": sorted(step_ms)[min(len(step_ms) - 1, len(step_ms) * 9 // 10)],
                               "e2e_median": e2e_med, "e2e_p10": e2e_stats[1], "e2e_p90": e2e_stats[2],
                               "e2e_cold_first_call": e2e_stats[3], "enum_ms_avg": enum_avg_ms,
                               "phases_device_median": phase_med},
            # (combination x input state) costs C(u, s) the search minimises over, per
            # second; each combination is enumerated once per type and
            # its D_in input states enter through the per-prefix cross-term fold
            "evals_per_s": info.evals / (ms_per_step * 1e-3),
            "e2e": {"value": combos / (e2e_med * 1e-3), "unit": UNIT,
                    "h2d_bytes_per_step": problem_bytes(prob), "d2h_bytes_per_step": plan_bytes(prob),
                    "plan_search_ms": e2e_med, "p10_ms": e2e_stats[1], "p90_ms": e2e_stats[2],
                    "cold_first_call_ms": e2e_stats[3],
                    "note": "ctx.search_plan(problem) from Python (marshalling included); calls alternate "
                            "between two problems of the same structure with different values, so every "
                            "call uploads its tables and recomputes the whole path; the structure's host "
                            "schedule / device buffers are reused (warm). cold_first_call_ms: a fresh "
                            "ctx's first call (prepare: validation, schedule, allocation, uploads)"},
            "gpu_launches": info.kernel_launches,
            "roofline": {"bound": "alu", "achieved": achieved_gops, "peak": peak, "unit": "Gop/s",
                         "frac": achieved_gops / peak, "traffic": traffic,
                         "frac_of_alu_only_peak": achieved_gops / peak_alu,
                         "note": "op = one fused add+min per strategy combination; peak = the measured "
                                 "rate of the loop's two-pipe group (N5 op 3: VIADDMNMX + 2 FMA-pipe IMAD "
                                 "+ VIMNMX3 per 3 combinations) or 64 VIADDMNMX lane-ops/clk/SM x 148 "
                                 "SMs x 1965 MHz, whichever is higher (DESIGN.md); achieved = combos / "
                                 "device time of the enumeration phase (all enum launches incl. the "
                                 "cross-term fold epilogue); traffic = DRAM bytes per enum launch from "
                                 "ncu (profiles/r02_ncu_enum_v9.json), algorithmic bytes ~0"},
            "intpipe_measured": {"op": "VIADDMNMX.U32", "lane_ops_per_s": ip_ops,
                                 "lane_ops_per_clk_per_sm": ip_ops / (SMS * 1e6 * (clocks["sm_mhz"] or 1965.0)),
                                 "frac_of_derived_peak": ip_ops / (peak_alu * 1e9),
                                 "two_pipe_group_addmin_per_s": ip3_ops,
                                 "two_pipe_per_clk_per_sm": ip3_ops / (SMS * 1e6 * (clocks["sm_mhz"] or 1965.0))},
            "clocks": clocks,
            "schedule": info.schedule,
            "plan_total_ns": plan.total_ns,
        }
        if minplus is not None:
            out["minplus_microbench"] = minplus
            best = max((r for r in minplus if r["dtype"] == "u32" and not r["argk"]), key=lambda r: r["addmin_per_s"])
            out["minplus_roofline"] = {
                "bound": "alu", "kernel": "minplus_tiled_kernel<u32>", "S": best["S"],
                "achieved": best["addmin_per_s"] / 1e9, "peak": peak_alu, "unit": "Gop/s",
                "frac": best["addmin_per_s"] / (peak_alu * 1e9),
                "note": "one fused add+min (VIADDMNMX.U32) per (i, j, k), S^3 per product; u64 add+min is "
                        "6 SASS instructions (IADD3, IADD3.X, 2 ISETP, 2 SEL), bound ~1/6 of this peak"}
        if world > 1:
            nr, nv = ctx.nccl_info()
            out["nccl"] = {"nranks": nr, "version": nv,
                           "collectives": "ncclAllReduce(ncclUint64, ncclMin) x 2 per step"}
    prep.close()
    ctx.close()
    return out


def run_cfp_mem(args, rank, world, local_rank):
    """Memory-constrained search on the config's graph:
    same metric (combos / device time of one full search), tables resident in
    HBM, L2 flushed between steps; e2e through cfp_search_plan_mem."""
    import numpy as np
    import torch

    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    from synth.memcfg import mem_workload
    if world > 1:
        raise SystemExit("--mem runs on one GPU (replicas only)")
    torch.cuda.set_device(local_rank)
    prob, quantum, limit = mem_workload(args.config, args.seed, args.dist)
    ctx = cfp.Context(device=local_rank)
    prep = ctx.prepare_mem(prob, quantum, limit)
    prep.time_kernels(True)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    for _ in range(args.warmup):
        flush_l2(torch, flush)
        torch.cuda.synchronize()
        prep.execute()
        prep.kernel_ms()
    plan0 = prep.fetch()
    enum_ms, tab_ms, step_ms = [], [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            flush_l2(torch, flush)
            torch.cuda.synchronize()
            prep.execute()
            e, a, t, combos, launches = prep.kernel_ms()
            enum_ms.append(e)
            tab_ms.append(a)
            step_ms.append(t)
        torch.cuda.synchronize()
    plan = prep.fetch()
    assert plan.total_ns == plan0.total_ns and np.array_equal(plan.seg_index, plan0.seg_index)
    fold_ops = prep.fold_ops()
    clocks = clk.summary()
    # e2e through cfp_search_plan_mem, alternating two value sets of one
    # structure (every call uploads values; K0 / T / enumeration / DP rerun)
    probs, want = [prob, perturbed(prob)], [plan0.total_ns, None]
    e2e = []
    for i in range(args.warmup + max(6, min(args.steps, 20))):
        t0 = time.perf_counter()
        p2 = ctx.search_plan_mem(probs[i % 2], quantum, limit)
        dt = (time.perf_counter() - t0) * 1e3
        if want[i % 2] is None:
            want[i % 2] = p2.total_ns
        assert p2.total_ns == want[i % 2]
        if i >= args.warmup:
            e2e.append(dt)
    t0 = time.perf_counter()
    c2 = cfp.Context(device=local_rank)
    t1 = time.perf_counter()
    c2.search_plan_mem(prob, quantum, limit)
    cold_ms = (time.perf_counter() - t1) * 1e3
    c2.close()
    del t0
    ms = statistics.median(step_ms)
    e_ms = statistics.median(enum_ms)
    f_ms = statistics.median(tab_ms) - e_ms
    peak_alu = alu_peak_gops(1965.0)
    # the enumeration body runs on two pipes (2 VIADDMNMX + 2 FMA-pipe adds + 1
    # VIMNMX3 per 4 combinations): peak = the measured two-pipe rate (N5 op 3)
    ip3_ops, _ = ctx.intpipe_bench(3, 4000)
    peak = max(peak_alu, ip3_ops / 1e9)
    achieved = combos / (e_ms * 1e-3) / 1e9
    mem_bytes = sum(0 if t.mem is None else t.mem.nbytes for t in prob.types)
    out = {
        "metric": METRIC, "value": combos / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{args.config} memory-constrained search (NEXT-1, Eq. 4): {args.dist} "
                               f"tables seed {args.seed}, quantum {quantum} KiB, limit {limit} KiB "
                               f"(Qmax {limit // quantum})",
                   "combos_per_step": combos, "l2": "flushed (512 MiB write) between timed steps"},
        "plan_search_ms": {"device_median": ms, "enum_ms": e_ms, "fold_and_minima_ms": f_ms,
                           "a0_and_chain_argmin_plan_ms": ms - e_ms - f_ms, "e2e_median": statistics.median(e2e),
                           "e2e_cold_first_call": cold_ms},
        "e2e": {"value": combos / (statistics.median(e2e) * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": problem_bytes(prob) + mem_bytes, "d2h_bytes_per_step":
                plan_bytes(prob) + 8 * len(prob.instances)},
        "gpu_launches": launches,
        "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Gop/s",
                     "frac": achieved / peak, "traffic": ncu_traffic("r02_ncu_mem_v9", "mem_enum_kernel<unsigned int, 4>"),
                     "frac_of_alu_only_peak": achieved / peak_alu,
                     "note": "enumeration kernels: one fused add+min per strategy combination "
                             "(K0[p] + T[ctx][sigma] into its (layout, memory) class), the 16-byte body on "
                             "two pipes; peak = max(N5 op-3 two-pipe rate, 64 VIADDMNMX/clk/SM); traffic: "
                             "DRAM bytes of one layer-type launch (profiles/r02_ncu_mem_v9.json)"},
        "fold_roofline": {"bound": "alu", "achieved": fold_ops / (f_ms * 1e-3) / 1e9, "peak": peak_alu,
                          "unit": "Gop/s", "frac": fold_ops / (f_ms * 1e-3) / 1e9 / peak_alu,
                          "addmins_per_step": fold_ops},
        "clocks": clocks, "plan_total_ns": plan.total_ns, "plan_total_q": plan.total_q,
        "quantisation": mem_slack(prob, plan, quantum, limit),
    }
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline_mem(prob, quantum)
    prep.close()
    ctx.close()
    return out


def hbm_peak_gbs() -> Tuple[float, str]:
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs (copy, read+write)"
    except Exception:
        return 7700.0, "fallback: B200_PROFILING.md nominal 7.7 TB/s"


def run_cfp_dense(args, rank, world, local_rank):
    """Dense per-plan tables: the config's
    graph with one profiled time per whole-segment plan, generated on the
    device (synth.generators.dense_table stream); the tables (C3: 2 x 18.3 GB)
    are streamed once per search.  Roofline: HBM bytes of the table stream."""
    import numpy as np
    import torch

    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    from synth import generators as G
    if world > 1:
        raise SystemExit("--dense runs on one GPU")
    torch.cuda.set_device(local_rank)
    prob = G.make_config(args.config, args.seed, args.dist)
    ctx = cfp.Context(device=local_rank)
    used = sorted({prob.transitions[int(t)].type for t in prob.instances})
    bufs = {}
    for t in used:
        n = prob.num_combinations(t)
        bufs[t] = torch.empty(n, dtype=torch.int32, device="cuda")
        ctx.dense_fill(bufs[t].data_ptr(), n, G.dense_base(args.seed, t))
    ptrs = [bufs[t].data_ptr() if t in bufs else 0 for t in range(len(prob.types))]
    prep = ctx.prepare_dense(prob, ptrs)
    prep.time_kernels(True)
    for _ in range(args.warmup):
        prep.execute()
        prep.kernel_ms()
    plan0 = prep.fetch()
    s_ms, t_ms = [], []
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()          # tables >> L2 (126 MB): no flush needed
            prep.execute()
            a, t, combos, nbytes, launches = prep.kernel_ms()
            s_ms.append(a)
            t_ms.append(t)
        torch.cuda.synchronize()
    plan = prep.fetch()
    assert plan.total_ns == plan0.total_ns and np.array_equal(plan.seg_index, plan0.seg_index)
    clocks = clk.summary()
    e2e = []
    for i in range(args.warmup + max(3, min(args.steps, 10))):
        t0 = time.perf_counter()
        p2 = ctx.search_plan_dense(prob, ptrs)
        dt = (time.perf_counter() - t0) * 1e3
        if i >= args.warmup:
            e2e.append(dt)
    assert p2.total_ns == plan0.total_ns
    ms = statistics.median(t_ms)
    sm = statistics.median(s_ms)
    peak, peak_src = hbm_peak_gbs()
    achieved = nbytes / (sm * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": combos / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{args.config} with dense per-plan tables (NEXT-2, P:572-574): one hashed "
                               f"24-bit time per whole-segment plan (seed {args.seed}), {nbytes / 1e9:.1f} GB "
                               f"of tables resident in HBM",
                   "combos_per_step": combos, "l2": "tables >> L2: every step streams them from HBM"},
        "plan_search_ms": {"device_median": ms, "table_stream_ms": sm, "e2e_median": statistics.median(e2e)},
        "e2e": {"value": combos / (statistics.median(e2e) * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": problem_bytes(prob), "d2h_bytes_per_step": plan_bytes(prob),
                "note": "tables are device-resident inputs (tens of GB); e2e covers the search call"},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": ncu_traffic("r02_ncu_dense_v8", "dense_rows"),
                     "note": f"dense_rows_kernel: 4 B read per combination (algorithmic) / stream time; "
                             f"traffic: DRAM bytes of one layer-type launch (profiles/r02_ncu_dense_v8.json); "
                             f"peak: {peak_src}"},
        "clocks": clocks, "plan_total_ns": plan.total_ns,
    }
    prep.close()
    ctx.close()
    return out


def run_cfp_budget(args, rank, world, local_rank):
    """Dynamic profiling budget: every whole-segment
    plan task of the config's used types screened in index order against
    f x best (f = 2) over the dense per-plan tables of NEXT-2 (device
    generator), one scan per type.  Roofline: HBM, 4 B read per task."""
    import torch

    from paper_2504_00598_b200 import build as B
    B.build()
    from paper_2504_00598_b200 import cfp
    from synth import generators as G
    if world > 1:
        raise SystemExit("--budget runs on one GPU")
    torch.cuda.set_device(local_rank)
    prob = G.make_config(args.config, args.seed, args.dist)
    ctx = cfp.Context(device=local_rank)
    used = sorted({prob.transitions[int(t)].type for t in prob.instances})
    bufs, ns = {}, {}
    for t in used:
        ns[t] = prob.num_combinations(t)
        bufs[t] = torch.empty(ns[t] + 8, dtype=torch.int32, device="cuda")
        ctx.dense_fill(bufs[t].data_ptr(), ns[t], G.dense_base(args.seed, t))
    num, den = 2, 1
    tasks = float(sum(ns.values()))

    def step():
        res, ms = {}, 0.0
        for t in used:
            r, k = ctx.profile_budget(bufs[t].data_ptr(), ns[t], num, den, timed=True)
            res[t] = r
            ms += k
        return res, ms

    for _ in range(args.warmup):
        ref, _ = step()
    k_ms, big_ms, e2e = [], [], []
    big = max(used, key=lambda t: ns[t])
    with ClockSampler(local_rank) as clk:
        for _ in range(args.steps):
            torch.cuda.synchronize()          # tables >> L2: every step streams them from HBM
            t0 = time.perf_counter()
            res, ms = step()
            e2e.append((time.perf_counter() - t0) * 1e3)
            assert res == ref
            k_ms.append(ms)
            _, kb = ctx.profile_budget(bufs[big].data_ptr(), ns[big], num, den, timed=True)
            big_ms.append(kb)
        torch.cuda.synchronize()
    clocks = clk.summary()
    ms = statistics.median(k_ms)
    kb = statistics.median(big_ms)
    peak, peak_src = hbm_peak_gbs()
    achieved = ns[big] * 4 / (kb * 1e-3) / 1e9
    pruned = sum(r["pruned"] for r in ref.values())
    traffic = ncu_traffic("r02_ncu_budget_v8", "budget_kernel")
    out = {
        "metric": "budgeted profiling tasks screened/sec (dense per-plan tables, NEXT-3)",
        "value": tasks / (ms * 1e-3), "unit": "tasks/s", "n_gpus": 1, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u32", "data": "synthetic",
        "config": {"workload": f"{args.config} dense per-plan tables (seed {args.seed}), every plan task of "
                               f"the {len(used)} used types screened against f x best, f = {num}/{den}",
                   "tasks_per_step": tasks, "l2": "tables >> L2: every step streams them from HBM"},
        "budget": {"pruned": pruned, "infeasible": sum(r["infeasible"] for r in ref.values()),
                   "spent_ns": sum(r["spent"] for r in ref.values()),
                   "full_ns": sum(r["full"] for r in ref.values())},
        "e2e": {"value": tasks / (statistics.median(e2e) * 1e-3), "unit": "tasks/s",
                "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 64 * len(used),
                "note": "tables are device-resident inputs (tens of GB); e2e = host wall time of the calls"},
        "gpu_launches": len(used),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic,
                     "note": f"budget_kernel on the largest type ({ns[big]} tasks): 4 B read per task "
                             f"(algorithmic, {ns[big] * 4} B per launch) / device time of the call; "
                             f"traffic = DRAM bytes of that launch (profiles/r02_ncu_budget_v8.json); "
                             f"peak: {peak_src}"},
        "clocks": clocks,
    }
    if not args.no_cpu_baseline:
        from oracle import profiling as PR
        m = 1 << 24
        W = G.dense_table(args.seed, big, m)
        t0 = time.perf_counter()
        PR.budget(W, num, den)
        dt = time.perf_counter() - t0
        out["cpu_baseline"] = {"value": m / dt, "unit": "tasks/s", "cores": 1, "kind": "oracle",
                               "sample": f"first {m} tasks of type {big} (numpy prefix-minimum oracle, "
                                         f"{dt:.2f} s)"}
    ctx.close()
    return out


def spawn_ranks(args):
    """`bench.py --gpus N` without a launcher: start N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and exit with their status.
    Fails loudly when fewer than N GPUs are visible (the reference arm is the
    CPU oracle and runs on rank 0 alone, so it needs no GPU)."""
    import socket
    if args.impl != "reference":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            sys.exit(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible; "
                     f"not reporting a {n}-GPU number as {args.gpus}")
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cfp", choices=["cfp", "reference"])
    ap.add_argument("--config", default="C3")
    ap.add_argument("--dist", default="shaped")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-minplus", action="store_true", help="skip the (min,+) product microbenchmark")
    ap.add_argument("--mem", action="store_true", help="memory-constrained search (NEXT-1) instead")
    ap.add_argument("--dense", action="store_true", help="dense per-plan tables (NEXT-2) instead")
    ap.add_argument("--budget", action="store_true", help="dynamic profiling budget (NEXT-3) instead")
    args = ap.parse_args()
    if args.gpus < 1:
        sys.exit("bench.py: --gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        spawn_ranks(args)                      # re-exec under torchrun, one rank per GPU
        return
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        sys.exit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: refusing to report a line "
                 f"whose n_gpus differs from the request")
    if world > 1 and (args.mem or args.dense or args.budget):
        sys.exit("bench.py: --mem / --dense / --budget are single-GPU paths (DESIGN.md §8); use --gpus 1")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.warmup < 3:
        args.warmup = 3
    from synth import make_config
    prob = make_config(args.config, args.seed, args.dist)
    if args.impl == "reference":
        out = run_reference(args, prob, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if args.mem:
        print(json.dumps(run_cfp_mem(args, rank, world, local_rank)), flush=True)
        return
    if args.dense:
        print(json.dumps(run_cfp_dense(args, rank, world, local_rank)), flush=True)
        return
    if args.budget:
        print(json.dumps(run_cfp_budget(args, rank, world, local_rank)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_cfp(args, prob, rank, world, local_rank)
    if out is not None and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(prob)
    if out is not None:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
