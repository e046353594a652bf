#!/usr/bin/env python
"""bench.py — throughput of the MRAB / SBP-SAT overset hot path on B200.

Contract:
  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl mrab|reference] [--config C]
One "step" = one MRAB macro step H = S_max h of the whole hot path (every mesh's fused
SBP-SAT RHS + AB update at its own rate, donor intermediate states, Lagrange gathers) on
BASELINE.json configs[3] (config 4, full size: the largest configuration that fits one GPU,
23.9 M points; BASELINE.json's metric names no config) unless --config says otherwise; the
cylinder stand-in (config 3) is measured beside it as `secondary`.
metric = grid-point RHS evaluations per second (sum over meshes of active points x RHS
evaluations, fp64).  L2 is scrubbed (256 MiB write + 256 MiB read of another buffer)
between timed steps.  Multi-GPU: one
process per GPU, each an independent replica (no data-path collective).
--impl reference times the oracle (oracle/, plain numpy fp64) on host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

os.environ.setdefault("OMP_NUM_THREADS", "1")       # the oracle baseline is single-threaded
ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "grid-point RHS evals/sec (fp64)"
UNIT = "point-RHS/s"
FALLBACK_HBM = 6650.0
# oracle sample scale per config: configs 4 and 5 at full size need > 15 min of oracle overset
# setup alone, so their CPU sample is the same workload at the reduced "test" size (identical
# per-point arithmetic, smaller meshes)
ORACLE_SCALE = {1: "full", 2: "full", 3: "full", 4: "test", 5: "test"}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _fp64_peak():
    """FP64 DFMA throughput measured on this pool's B200 by scripts/probes/fp64_probe.cu."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "r01", "fp64_probe.json")))
        return float(d["fp64_dfma_tflops"]), "measured (profiles/r01/fp64_probe.json)"
    except Exception:
        return None, "unavailable"


def _cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.strip()]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def combine_ranks(total_ms, point_rhs, dist=None, device="cpu"):
    """Whole-job numbers over replicas: the MAX of the ranks' timed totals and
    the SUM of their point-RHS counts (value = sum / max)."""
    if dist is None:
        return total_ms, point_rhs
    import torch
    t = torch.tensor([total_ms], device=device, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    c = torch.tensor([float(point_rhs)], device=device, dtype=torch.float64)
    dist.all_reduce(c, op=dist.ReduceOp.SUM)
    return float(t.item()), int(c.item())


def _problem(cid, scale, sr=None):
    import synth
    kw = {} if sr is None else {"sr": sr}
    return synth.make_config(cid, scale, **kw)


_ORACLE = {}


def _oracle_problem(cid):
    return _problem(cid, ORACLE_SCALE[cid])


def _oracle_worker(args):
    cid, n_macro, budget_s = args
    os.environ["OMP_NUM_THREADS"] = "1"
    return _oracle_sample(_oracle_problem(cid), n_macro, budget_s)


def _oracle_cores(cid, budget_s):
    """Oracle throughput on 1 host core and on every host core (os.cpu_count() independent
    single-threaded oracle processes running the same bounded sample at once; the aggregate
    is the sum of their point-RHS over the longest of their times)."""
    import multiprocessing as mp
    n = os.cpu_count() or 1
    pr1, dt1, n1 = _oracle_sample(_oracle_problem(cid), 1000, budget_s)
    ctx = mp.get_context("spawn")
    with ctx.Pool(n) as pool:
        res = pool.map(_oracle_worker, [(cid, n1, 1e9)] * n)
    pr_all = sum(r[0] for r in res)
    dt_all = max(r[1] for r in res)
    return {"value_1_core": pr1 / dt1, "seconds_1_core": dt1, "macro_steps": n1,
            "value_all_cores": pr_all / dt_all, "cores_all": n, "seconds_all_cores": dt_all}


def _oracle_sample(p, n_macro, budget_s):
    """Oracle (plain numpy fp64, oracle/) timed on host cores: `n_macro` macro steps of the
    same workload from a synthetic full history (rings = m copies of R(q0); the arithmetic
    of a step is identical).  Returns (point_rhs, seconds, macro steps done)."""
    from oracle import timeint, rhs as orhs
    if id(p) not in _ORACLE:
        setup = orhs.build(p)
        mr = timeint.MRAB(p, setup=setup)
        R0 = orhs.rhs(p, setup, mr.base)
        for g in range(len(p.meshes)):
            mr.rings[g] = [R0[g].copy() for _ in range(p.history_m)]
        _ORACLE[id(p)] = (setup, mr)
    setup, mr = _ORACLE[id(p)]
    active = [int(setup.geom[g].active.sum()) for g in range(len(p.meshes))]
    c0 = list(mr.counts)
    t0 = time.perf_counter()
    done = 0
    while done < n_macro:
        mr.macro_step()
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    pr = sum((mr.counts[g] - c0[g]) * active[g] for g in range(len(p.meshes)))
    return pr, dt, done


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return 0
    p = _oracle_problem(args.config)
    per_step, tot_pr, tot_t = [], 0, 0.0
    for it in range(args.warmup + args.steps):
        pr, dt, _ = _oracle_sample(p, 1, 1e9)
        if it >= args.warmup:
            tot_pr += pr
            tot_t += dt
            per_step.append(dt)
    value = tot_pr / tot_t
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * tot_t / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": p.notes["workload"], "config": args.config,
                   "l2": "n/a (host)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "cpu_model": _cpu_model(),
                         "sample": f"{args.steps} oracle MRAB macro steps of config "
                                   f"{args.config} at {ORACLE_SCALE[args.config]} size "
                                   f"({p.notes['workload']}) from a synthetic history"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def _secondary(cid, args, stream, l2_flush):
    """The cylinder stand-in (config 3) measured beside the contract line: value, step time and
    the roofline fraction of its dominant kernel (same timing rules)."""
    import torch
    from paper_1805_06607_b200 import mrab
    p = _problem(cid, "full")
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    G = len(p.meshes)
    ctx.step(p.history_m - 1)
    for _ in range(max(args.warmup, 3)):
        ctx.step(1)
    torch.cuda.synchronize()
    ev0, _, _ = ctx.counters()
    k_steps = max(args.steps, 20)
    tot = 0.0
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(k_steps):
        l2_flush(k)
        a0.record(stream)
        ctx.step(1)
        a1.record(stream)
        torch.cuda.synchronize()
        tot += a0.elapsed_time(a1)
    ev1, _, _ = ctx.counters()
    active = [plan.info(g)[1] for g in range(G)]
    pr = sum((ev1[g] - ev0[g]) * active[g] for g in range(G))
    per = []
    for g in range(G):
        ms, by = ctx.time_kernel(0, g, reps=20, flush_l2=True)
        per.append((by * (ev1[g] - ev0[g]) / k_steps, ms, by, g))
    _, ms, by, gdom = max(per)
    peak, _ = _peaks()
    ctx.close()
    return {"config": cid, "workload": p.notes["workload"], "value": pr / (tot * 1e-3),
            "unit": UNIT, "ms_per_step": tot / k_steps, "steps": k_steps,
            "roofline": {"kernel": f"k_rhs2d on mesh {gdom} ({p.meshes[gdom].name})",
                         "achieved": by / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                         "frac": by / (ms * 1e-3) / 1e9 / peak, "ms_per_launch": ms,
                         "algorithmic_bytes_per_launch": by}}


def run_gpu(args):
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    from paper_1805_06607_b200 import mrab

    p = _problem(args.config, "full", args.sr)
    plan = mrab.Plan(p)
    ctx = mrab.Context(plan, p.q0)
    part = None
    if ws > 1 and args.dist:
        # one problem over the ranks: meshes partitioned by work, donor data over NCCL
        owner, load = mrab.partition(plan, ws)
        ctx.attach_nccl(dist, owner)
        part = {"owner": owner, "load": load}
        args.no_srab = args.no_secondary = True
    stream = torch.cuda.current_stream()
    G = len(p.meshes)
    nboot = p.history_m - 1

    # bootstrap (untimed for `value`, reported)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    ctx.step(nboot)
    e1.record(stream)
    torch.cuda.synchronize()
    boot_ms = e0.elapsed_time(e1)
    for _ in range(args.warmup):
        ctx.step(1)
    torch.cuda.synchronize()

    # L2 flush between timed steps: write 256 MiB, then read another 256 MiB so the L2 holds
    # clean lines of an unrelated buffer (a write-only flush would leave ~126 MB of dirty
    # lines whose write-back would be charged to the next timed step).
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    scrub = torch.ones(32 << 20, dtype=torch.float64, device="cuda")

    def l2_flush(k):
        flush.fill_(k & 0xff)
        scrub.sum()
    ev0, _, _ = ctx.counters()
    clocks = Clocks(local)
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    time.sleep(0.25)
    total_ms = 0.0
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    for k in range(args.steps):
        l2_flush(k)                                 # outside the timed events
        starts[k].record(stream)
        ctx.step(1)
        ends[k].record(stream)
    torch.cuda.synchronize()
    clk = clocks.stop()
    if dist is not None:
        dist.barrier()
    for k in range(args.steps):
        total_ms += starts[k].elapsed_time(ends[k])
    ev1, _, _ = ctx.counters()
    active = [plan.info(g)[1] for g in range(G)]
    pr = int(sum((ev1[g] - ev0[g]) * active[g] for g in range(G)))
    t_max, pr_sum = combine_ranks(total_ms, pr, dist, "cuda")
    value = pr_sum / (t_max * 1e-3)
    launches = ctx.launches_per_macro_step()

    # ---- roofline of the dominant kernel (live CUDA-event timing, L2 flushed) ----------
    peak, peak_src = _peaks()
    per_mesh = []
    evals_per_step = [(ev1[g] - ev0[g]) / args.steps for g in range(G)]
    # the dominant (HBM-bound) kernel is the mesh RHS that moves the most algorithmic bytes
    # per macro step; meshes whose whole working set stays in L2 across their substeps (the
    # config-3 O-grid: 13 MB per launch, four launches back to back) are latency-bound and
    # reported beside it with their warm (in-step) launch time
    for g in range(G):
        ms, by = ctx.time_kernel(0, g, reps=20, flush_l2=True)
        per_mesh.append((by * evals_per_step[g], ms, by, g))
    _, ms, by, gdom = max(per_mesh)
    achieved = by / (ms * 1e-3) / 1e9
    others = []
    for bpstep, msg, byg, g in per_mesh:
        if g == gdom:
            continue
        msw, _ = ctx.time_kernel(0, g, reps=20, flush_l2=False)
        others.append({"kernel": f"k_rhs on mesh {g} ({p.meshes[g].name})", "bound": "latency (L2-resident)",
                       "launches_per_step": evals_per_step[g], "ms_per_launch_warm": msw,
                       "ms_per_launch_cold": msg, "algorithmic_bytes_per_launch": byg})
    kernel_times = {}
    for kid, name in ((0, "k_rhs"), (1, "k_visc"), (2, "k_interp")):
        if kid == 1 and (not p.viscous or p.dim != 3):
            continue
        tot = 0.0
        for g in range(G):
            mk, _ = ctx.time_kernel(kid, g, reps=10, flush_l2=True)
            tot += mk * evals_per_step[g]
        kernel_times[name] = tot
    traffic = None
    fp64_pct = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        ent = tj.get(f"config{args.config}/mesh{gdom}/k_rhs2d" if p.dim == 2
                     else f"config{args.config}/mesh{gdom}/k_rhs3d")
        if ent:
            traffic = ent["total"]
            fp64_pct = ent.get("fp64_pipe_pct")
    except Exception:
        traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic,
            "kernel": (f"k_rhs2d (fused RHS+SAT+AB) on mesh {gdom} ({p.meshes[gdom].name})" if p.dim == 2 else
                       (f"k_rhs3z (fused one-pass RHS + SAT + AB, z-marching) on mesh {gdom} ({p.meshes[gdom].name})"
                        if os.environ.get("MRAB_3D_FUSED", "0") not in ("", "0") else
                        f"k_flux3w + k_div3w (RHS in two passes on 16x8x4 tiles, SAT, AB) on mesh {gdom} ({p.meshes[gdom].name})")),
            "algorithmic_bytes_per_launch": by, "ms_per_launch": ms, "peak_source": peak_src,
            "kernel_ms_per_step_cold": kernel_times, "other_meshes": others,
            "fp64_pipe_pct_ncu": fp64_pct, "fp64_peak_tflops": _fp64_peak()[0],
            "fp64_peak_source": _fp64_peak()[1]}

    # ---- end to end through the C ABI with host buffers --------------------------------
    host = [torch.empty(q.shape, dtype=torch.float64).pin_memory() for q in p.q0]
    for g in range(G):
        ctx.get_state(g, out=host[g])
    nbytes = int(sum(h.numel() * 8 for h in host))
    ke = max(3, min(args.steps, 50))
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ev0e, _, _ = ctx.counters()
    t0.record(stream)
    for _ in range(ke):
        for g in range(G):
            ctx.set_state(g, host[g])
        ctx.step(1)
        for g in range(G):
            ctx.get_state(g, out=host[g])
    t1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = t0.elapsed_time(t1)
    ev1e, _, _ = ctx.counters()
    pr_e = sum((ev1e[g] - ev0e[g]) * active[g] for g in range(G))
    e2e = {"value": pr_e / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": nbytes,
           "d2h_bytes_per_step": nbytes, "steps": ke}

    # ---- MRAB vs single-rate AB wall time (same simulated time) ------------------------
    srab = None
    if rank == 0 and not args.no_srab:
        plan_s = mrab.Plan(p, steps=[1] * G)
        ctx_s = mrab.Context(plan_s, p.q0)
        ctx_s.step(nboot)
        for _ in range(3):
            ctx_s.step(1)
        S = p.s_max
        ks = max(S * 4, (min(args.steps, 50) // 1) * S)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tot_s = 0.0
        for k in range(ks):
            l2_flush(k)
            a0.record(stream)
            ctx_s.step(1)
            a1.record(stream)
            torch.cuda.synchronize()
            tot_s += a0.elapsed_time(a1)
        srab_ms_per_H = tot_s / ks * S
        mrab_ms_per_H = total_ms / args.steps
        srab = {"mrab_ms_per_macro_step": mrab_ms_per_H, "srab_ms_per_same_time": srab_ms_per_H,
                "saving": 1.0 - mrab_ms_per_H / srab_ms_per_H,
                "predicted_work_ratio_mrab_over_srab":
                    sum(active[g] * S / p.meshes[g].step_multiple for g in range(G)) /
                    (S * sum(active))}
        ctx_s.close()

    secondary = None
    if rank == 0 and args.config != 3 and not args.no_secondary:
        ctx.close()
        secondary = _secondary(3, args, stream, l2_flush)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        oc = _oracle_cores(args.config, 15.0)
        po = _oracle_problem(args.config)
        cpu = {"value": oc["value_all_cores"], "unit": UNIT, "cores": oc["cores_all"],
               "kind": "oracle", "cpu_model": _cpu_model(),
               "value_1_core": oc["value_1_core"],
               "sample": f"{oc['macro_steps']} oracle MRAB macro step(s) of config {args.config} at "
                         f"{ORACLE_SCALE[args.config]} size ({po.notes['workload']}) from a "
                         f"synthetic history, in each of {oc['cores_all']} independent "
                         f"single-threaded processes at once ({oc['seconds_all_cores']:.1f} s); "
                         f"1 process alone: {oc['seconds_1_core']:.1f} s"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if part else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": p.notes["workload"], "config": args.config,
                       "order_n": p.order_n, "history_m": p.history_m,
                       "step_multiples": [m.step_multiple for m in p.meshes],
                       "points": [plan.info(g)[0] for g in range(G)],
                       "active_points": active, "l2": "flushed between timed steps (256 MiB)",
                       "parallelism": (f"mesh partition x{ws} (owner {part['owner']}, donor data over NCCL)" if part
                                       else (f"replicas x{ws}" if ws > 1 else "1 GPU"))},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": int(launches * args.steps), "launches_per_step": launches,
            "clocks": clk, "bootstrap_ms": boot_ms, "mrab_vs_srab": srab,
            "secondary": secondary,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist is not None:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="mrab", choices=["mrab", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--sr", type=int, default=None)
    ap.add_argument("--no-srab", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-secondary", action="store_true")
    ap.add_argument("--dist", action="store_true",
                    help="N > 1: partition the meshes of ONE problem over the ranks (strong scaling) "
                         "instead of independent replicas")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
