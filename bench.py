#!/usr/bin/env python
"""Benchmark: subgraphs enumerated per second on B200 (BASELINE.json metric).

Workload (a "step"): one full k-clique count of BASELINE config 3 — the
Chung-Lu power-law graph with 100,000 vertices / 947,479 edges (SURVEY §8(d)
recipe, seed 3) — through ``run_clique`` (clique_app pipeline) in ``opt`` mode
(on-device load balancer on).  Default k=8 (9,384,222,498 cliques).  Counts
are checked against the pinned golden value every step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--k 8]
  python bench.py --impl reference ...   # CPU restatement of the reference

Multi-GPU: launched by torchrun, one process per GPU; rank r takes the
cyclic share r (mod N) of the cost-sorted root tasks (no data-path
collective); counts meet in ONE all_reduce; time = max over ranks.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "subgraphs enumerated/sec (k-clique, k-motif) at 1/2/4/8 B200 vs CPU ref"
UNIT = "subgraphs/s"


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def golden_counts():
    try:
        with open(os.path.join(ROOT, "tests", "golden", "scale_golden.json")) as fh:
            return json.load(fh).get("cfg3", {}).get("clique", {})
    except Exception:
        return {}


def ncu_traffic(k):
    """dram bytes per launch of the enumeration kernel from the committed
    ncu --set full capture (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("clique_enum_kernel", {}).get("k%d" % k)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for nm, flag in zip(names, parts[3:7]):
                if flag.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return None
        load = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(load), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    return rank, world


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_sample(g, k, budget_s, seed=0):
    """Reference algorithm (oracle/ C restatement of engine.run's clique
    pipeline, id order) on all host cores over a seeded random root order,
    time-boxed.  Returns (rate, leaves, seconds, roots_done, threads)."""
    import numpy as np
    import oracle
    threads = os.cpu_count() or 1
    roots = np.random.default_rng(seed).permutation(g.n).astype(np.int64)
    t0 = time.perf_counter()
    r = oracle.clique_run(g, k, roots=roots, threads=threads, time_budget_s=budget_s)
    dt = time.perf_counter() - t0
    return r["leaves"] / dt, r["leaves"], dt, r["roots_done"], threads


def run_reference(args):
    rank, world = dist_setup()
    if rank != 0:
        return 0
    from paper_2212_04551_b200 import synth
    g = synth.config_graph("cfg3")
    per = max(2.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_sample(g, args.k, per, seed=1000 + _)
    rates, leaves, secs, roots = [], 0, 0.0, 0
    for i in range(args.steps):
        rate, lv, dt, rd, threads = cpu_sample(g, args.k, per, seed=i)
        rates.append(rate)
        leaves += lv
        secs += dt
        roots += rd
    value = leaves / secs if secs > 0 else 0.0
    sample = ("each step: reference clique_app pipeline (oracle/wm_oracle.c restatement of "
              "engine.py:214-241, id order) over a seeded random permutation of the %d roots, "
              "time-boxed to %.0f s; %d roots completed over %d steps" % (g.n, per, roots, args.steps))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(1, args.steps),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32/u64",
        "data": "synthetic", "config": workload_config(g, args.k, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": sample, "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_config(g, k, world):
    return {"workload": "cfg3 k-clique counting, k=%d, Chung-Lu power-law n=%d m=%d (gamma 2.3, "
                        "seed 3)" % (k, g.n, g.m),
            "k": k, "app": "clique_app", "graph": "chung_lu(100000, 1000000, 2.3, seed=3)",
            "n": g.n, "m": g.m, "order": "degree", "mode": "opt",
            "parallelism": "roots sharded cyclically over %d GPU(s)" % world,
            "l2": "flushed between timed steps (256 MiB write)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)

    rank, world = dist_setup()
    import numpy as np
    import torch
    from paper_2212_04551_b200 import BalanceConfig, engine, run_clique, synth
    from paper_2212_04551_b200.graph import CsrGraph
    dev = torch.cuda.current_device()
    g = synth.config_graph("cfg3")
    want = golden_counts().get(str(args.k), {}).get("count")
    shard = (rank, world)
    bc = BalanceConfig(threshold=1.0, poll_interval=32)
    stream = torch.cuda.current_stream()

    def step(graph):
        return run_clique(graph, args.k, mode="opt", balance_config=bc, shard=shard,
                          stream=stream, reduce=False)

    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.int32, device="cuda")
    for _ in range(args.warmup):
        r = step(g)
    # ---- timed: device-resident graph -------------------------------------
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    kern_ms, launches, results = [], 0, []
    clocks = ClockSampler(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks.start()
    for i in range(args.steps):
        flush.fill_(i)  # L2 flush, outside the event pair
        ev[i][0].record(stream)
        r = step(g)
        ev[i][1].record(stream)
        kern_ms.append(r.kernel_ms)
        launches += r.launches
        results.append(r)
    torch.cuda.synchronize()
    clk = clocks.stop()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    total_ms = sum(step_ms)
    if world > 1:
        torch.distributed.barrier()
        t = torch.tensor([total_ms, statistics.mean(kern_ms)], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        total_ms, kmean = t.tolist()
        cnt = torch.tensor([sum(x.clique_count for x in results)], dtype=torch.int64, device="cuda")
        torch.distributed.all_reduce(cnt)
        all_leaves = int(cnt.item())
    else:
        kmean = statistics.mean(kern_ms)
        all_leaves = sum(x.clique_count for x in results)
    per_step_count = all_leaves // args.steps
    value = all_leaves / (total_ms * 1e-3)

    # ---- e2e: host buffers through the public API, uploads inside ------------
    off_h = torch.from_numpy(np.asarray(g.offsets)).pin_memory()
    nbr_h = torch.from_numpy(np.asarray(g.neighbors_array)).pin_memory()
    e2e_ms, h2d, d2h, e2e_leaves = [], 0, 0, 0
    if world > 1:
        torch.distributed.barrier()
    for i in range(max(2, args.steps)):
        flush.fill_(i)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        gh = CsrGraph(g.n, off_h.numpy(), nbr_h.numpy())  # pinned host CSR, zero-copy view
        r = step(gh)                       # wm_graph_create (H2D) + wm_run + D2H of results
        engine.release_device_graph(gh)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        e2e_leaves += r.clique_count
        h2d = off_h.numel() * 8 + nbr_h.numel() * 4 + r.extra["h2d_bytes"]
        d2h = r.extra["d2h_bytes"]
    e2e_total = sum(e2e_ms)
    if world > 1:
        t = torch.tensor([e2e_total], dtype=torch.float64, device="cuda")
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_total = t.item()
        c = torch.tensor([e2e_leaves], dtype=torch.int64, device="cuda")
        torch.distributed.all_reduce(c)
        e2e_leaves = int(c.item())
    e2e_value = e2e_leaves / (e2e_total * 1e-3)

    if rank != 0:
        torch.distributed.barrier()
        return 0

    # ---- evidence (untimed): B_alg, LB off vs on, CPU baseline --------------
    peak, peak_src = load_peaks()
    rb = run_clique(g, args.k, count_bytes=True, stream=stream, shard=(0, 1))
    b_alg = rb.alg_bytes
    achieved = b_alg / (kmean * 1e-3) / 1e9 if world == 1 else None
    extras = {}
    if not args.no_extras:
        rw = run_clique(g, args.k, mode="wc", stream=stream, shard=(0, 1))
        ro = run_clique(g, args.k, mode="opt", balance_config=bc, stream=stream, shard=(0, 1))
        extras["load_balance"] = {
            "idle_warp_fraction_lb_off": rw.idle_warp_fraction,
            "idle_warp_fraction_lb_on": ro.idle_warp_fraction,
            "kernel_ms_lb_off": rw.kernel_ms, "kernel_ms_lb_on": ro.kernel_ms,
            "migrations": ro.migrations, "donations": ro.rebalance_count}
        extras["secondary"] = secondary_workloads(stream)
    cpu = None
    if world == 1 and args.cpu_budget > 0:
        rate, lv, dt, rd, threads = cpu_sample(g, args.k, args.cpu_budget)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
               "sample": "reference clique_app pipeline (oracle/wm_oracle.c restatement, id order) "
                         "on a seeded random root order of cfg3, time-boxed %.0f s: %d roots, %d "
                         "cliques in %.1f s" % (args.cpu_budget, rd, lv, dt),
               "cpu_model": cpu_model()}
    r0 = results[0]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32/u64", "data": "synthetic",
        "config": workload_config(g, args.k, world),
        "count_per_step": per_step_count,
        "count_matches_golden": (want is None) or (per_step_count == want),
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_total / len(e2e_ms)},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": (achieved / peak) if achieved else None,
                     "traffic": ncu_traffic(args.k), "peak_source": peak_src,
                     "kernel": "clique_enum_kernel<W=4>",
                     "alg_bytes_per_launch": b_alg,
                     "alg_bytes_def": "4 B x sum over productive search-tree nodes of "
                                      "deg+(last) in degree order (SURVEY 8(d))",
                     "kernel_ms": kmean},
        "cpu_baseline": cpu,
        "clocks": clk,
        "device": {"kernel_ms": kmean, "build_ms": r0.extra["build_ms"],
                   "device_ms": r0.device_ms, "warps": r0.warps,
                   "idle_warp_fraction": r0.idle_warp_fraction},
    }
    line.update(extras)
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.barrier()
    return 0


def secondary_workloads(stream):
    """configs 1 and 2 (exact, tiny) for the record; not the headline."""
    from paper_2212_04551_b200 import build_dictionary, run_clique, run_motifs, synth
    out = {}
    g1 = synth.config_graph("cfg1")
    for k in (3, 4):
        r = run_clique(g1, k, stream=stream, shard=(0, 1))
        out["cfg1_clique_k%d" % k] = {"count": r.clique_count, "kernel_ms": r.kernel_ms}
    from paper_2212_04551_b200 import BalanceConfig
    g2 = synth.config_graph("cfg2")
    lb = BalanceConfig(threshold=1.0, poll_interval=2)
    for k in (4, 6):
        for mode, kw in (("wc", {}), ("opt", {"balance_config": lb})):
            run_motifs(g2, k, build_dictionary(k), mode=mode, stream=stream, shard=(0, 1), **kw)
            r = run_motifs(g2, k, build_dictionary(k), mode=mode, stream=stream, shard=(0, 1), **kw)
            out["cfg2_motif_k%d%s" % (k, "" if mode == "wc" else "_opt")] = {
                "leaves": r.aggregated_total, "kernel_ms": r.kernel_ms,
                "subgraphs_per_s": r.subgraphs_per_second, "hist_head": r.pattern_counts[:6],
                "idle_warp_fraction": r.idle_warp_fraction}
    return out


if __name__ == "__main__":
    sys.exit(main())
