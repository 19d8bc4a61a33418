#!/usr/bin/env python
"""bench.py — throughput of the batched reduced-Hessian hot path on B200.

One *step* = one IPM-iteration-equivalent of the whole hot path
over every scenario the rank owns:
  pf_eval_constraints (A2/A3) → pf_jacobian (A4 Jacobian values + A5 LU
  refactorization) → pf_reduced_hessian_batch over ALL n_u directions (A6,
  A7.1–A7.5) → [all-gather of column slabs, direction mode only] →
  pf_condensed_kkt_solve_reg (A9: symmetrize + Σ_u + δ_w, FP64 Cholesky and
  solve, inside the paper's δ_w regularization loop, NEXT-3 — one trial when
  K_cond is positive definite).

Inputs (synth/, seeded): the paper's Table-1 shapes; λ is the
adjoint multiplier at each scenario's point (SURVEY §8(d) recipe:
G_xᵀλ = −∇_x(f + yᵀ[r; h])), computed before timing by pf_reduced_gradient
(NEXT-2) on the device (the reference arm: by the oracle).

Default workload (BASELINE.json configs[4], the north-star target):
case9241pegase-shaped synthetic grid, 8 load scenarios per GPU, scenario
sharding (weak scaling: N GPUs → 8N scenarios, no collective on the hot path).
`--config case1354|case2869|case118` runs the direction-sharded variants
(configs 1–3: one scenario, n_u columns split over ranks + one NCCL all-gather).

Metric (BASELINE.json): reduced-Hessian HVPs/sec (value) and condensed-KKT
factor+solve ms per IPM iteration (chol_ms_per_iter).  Timing: CUDA events on
the launching stream, L2 flushed (256 MiB write) before every step outside the
timed region, barrier + synchronize around the timed loop, max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "case9241x8": dict(grid="case9241", scen=8, mode="scenarios", baseline_cfg=4),
    "case2869": dict(grid="case2869", scen=1, mode="directions", baseline_cfg=3),
    "case1354": dict(grid="case1354", scen=1, mode="directions", baseline_cfg=2),
    "case118": dict(grid="case118", scen=1, mode="directions", baseline_cfg=1),
}
METRIC = "reduced-Hessian HVPs/sec and condensed-KKT factor+solve ms per IPM iteration"
# the δ_w loop of P:L1337–1342 (NEXT-3): start at 0, then 1e-8, ×10 up to 1e12
REG = dict(delta_init=0.0, delta_first=1e-8, growth=10.0, delta_max=1e12)
# FP64 peak of the Cholesky's DMMA pipe: MEASURED_PEAKS.json has no FP64 entry and the
# profiling guide states none, so the fallback is our own probe (tools/probe/fp64_peak.cu,
# profiles/r01_fp64_peak_probe.log: DMMA m8n8k4 37.18 TFLOP/s, DFMA 36.4)
FP64_PEAK_TFLOPS = 37.18
FP64_PEAK_SOURCE = "tools/probe/fp64_peak.cu on this pool's B200 (profiles/r01_fp64_peak_probe.log: DMMA m8n8k4)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="case9241x8", choices=list(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-generic", action="store_true", help="skip the dense-V generic-HVP timing")
    ap.add_argument("--no-next", action="store_true", help="skip the NEXT-row call timings")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    ap.add_argument("--profile-steps", type=int, default=0, help="run N untimed steps and exit (for ncu)")
    return ap.parse_args()


def env_rank():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def make_inputs(cfg, rank, world):
    """Seeded synthetic inputs of this rank (synth/ — no method arithmetic)."""
    from synth import make_scenario
    from synth.grid import table1_grid
    net, base = table1_grid(cfg["grid"])
    if cfg["mode"] == "scenarios":
        ids = list(range(rank * cfg["scen"], (rank + 1) * cfg["scen"]))
    else:
        ids = list(range(cfg["scen"]))
    pts = [base if s == 0 else make_scenario(net, base, s) for s in ids]
    return net, pts, ids


def read_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max(int(i.get("num_threads", 1)) for i in info) if info else 1
    except Exception:
        return os.cpu_count() or 1


def oracle_lambda(net, pt):
    """The oracle's adjoint multipliers at the point (the reference arm's λ)."""
    from oracle import pf_oracle as O
    part = O.partition(net)
    return O.adjoint_multipliers(net, part, pt, pt["y"])


def oracle_step(net, pt, lam):
    """The oracle (as it stands) for one scenario: constraints, Jacobians, K,
    the naive reduction, the condensed KKT δ_w loop (Cholesky) and solve.
    Returns (HVPs done, δ_w, Cholesky trials)."""
    import numpy as np
    from oracle import pf_oracle as O
    part = O.partition(net)
    O.constraints(net, pt)
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, lam, pt["y"], pt["sigma_s"], pt["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    Kc = O.condensed(0.5 * (Kh + Kh.T), pt["sigma_u"], 0.0)
    delta, trials, info, L = O.regularized_cholesky(Kc, **REG)
    if info == 0:
        O.chol_solve(L, np.ones(part["n_u"]))
    return part["n_u"], delta, trials


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    net, pts, _ = make_inputs(cfg, 0, 1)
    used = sorted({k % len(pts) for k in range(args.warmup + args.steps)})
    lams = {k: oracle_lambda(net, pts[k]) for k in used}   # inputs, before timing
    for k in range(args.warmup):
        oracle_step(net, pts[k % len(pts)], lams[k % len(pts)])
    t0 = time.perf_counter()
    hv, deltas, trials = 0, [], []
    for k in range(args.steps):
        n, d, t = oracle_step(net, pts[k % len(pts)], lams[k % len(pts)])
        hv += n
        deltas.append(d)
        trials.append(t)
    dt = time.perf_counter() - t0
    value = hv / dt
    cores = cpu_threads()
    sample = ("one %s-shaped scenario per step (all %d directions, naive-sensitivity oracle + the δ_w loop's dense "
              "Cholesky + solve)" % (cfg["grid"], hv // args.steps))
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "HVP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak" if cfg["mode"] == "scenarios" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s (BASELINE.json configs[%d])" % (args.config, cfg["baseline_cfg"]),
                       "grid": cfg["grid"], "n_b": net["n_b"], "n_l": net["n_l"], "n_g": net["n_g"],
                       "scenarios_per_gpu": cfg["scen"], "directions_per_step": hv // args.steps,
                       "lambda": "adjoint multipliers (oracle), before timing", "delta_w_max": max(deltas),
                       "reg_trials_max": max(trials), "parallelism": "CPU oracle, rank 0 only"},
            "cpu_baseline": {"value": value, "unit": "HVP/s", "cores": cores, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "HVP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    cfg = CONFIGS[args.config]
    rank, world, local = env_rank()
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2203_11875_b200 import Network, _build
    from paper_2203_11875_b200.dist import allgather_columns, column_partition
    if rank == 0:
        _build.build()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    f64 = torch.float64

    net, pts, ids = make_inputs(cfg, rank, world)
    S = len(pts)
    n_b, n_l, n_g = net["n_b"], net["n_l"], net["n_g"]
    if world > 1:
        dist.barrier()
    directions = cfg["mode"] == "directions"
    # ------------------------------------------------------------ handle
    tmp = Network(net, max_batch=1, max_scen=1, device=-1)
    n_u, n_x, m = tmp.dims["n_u"], tmp.dims["n_x"], tmp.dims["m"]
    tmp.close()
    # direction mode: tile-aligned column slabs, so every rank keeps the sparse-RHS reach lists
    tmp = Network(net, max_batch=-(-n_u // world), max_scen=S, device=-1)
    tile = tmp.dims["tile_cols"]
    tmp.close()
    col0, ncols, cpad = column_partition(n_u, world, rank, tile) if directions else (0, n_u, n_u)
    h = Network(net, max_batch=max(cpad, 1), max_scen=S, device=local, tile_cols=tile if directions else 0)
    h.profile(True)
    d = h.dims

    def stack(key):
        return np.ascontiguousarray(np.stack([np.asarray(p[key], dtype=np.float64) for p in pts]))

    host = {k: stack(k) for k in ("v", "theta", "p_g", "q_g", "p_d", "q_d", "lam", "y", "sigma_s", "sigma_x",
                                  "sigma_u")}
    host["rhs"] = np.ones((S, n_u))
    devt = {k: torch.as_tensor(a, device=dev) for k, a in host.items()}
    # λ: the adjoint multipliers at each scenario's point (NEXT-2 on the device), before timing
    h.pf_jacobian(S, devt["v"], devt["theta"])
    h.pf_reduced_gradient(S, devt["v"], devt["theta"], devt["p_g"], devt["y"], lam=devt["lam"], p_d=devt["p_d"])
    torch.cuda.synchronize()
    host["lam"] = devt["lam"].cpu().numpy()
    G = torch.empty(S, 2 * n_b, dtype=f64, device=dev)
    H = torch.empty(S, 2 * n_l, dtype=f64, device=dev)
    info_j = torch.empty(S, dtype=torch.int32, device=dev)
    KV = torch.empty(S, cpad, n_u, dtype=f64, device=dev)
    rhs = torch.empty(S, n_u, dtype=f64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    reg = {}

    def step(t, red_ev=None, chol_ev=None):
        rhs.copy_(t["rhs"])
        h.pf_eval_constraints(S, t["v"], t["theta"], t["p_g"], t["q_g"], t["p_d"], t["q_d"], G, H)
        if red_ev:
            red_ev[0].record(stream)
        h.pf_jacobian(S, t["v"], t["theta"], info=info_j)
        if ncols > 0:  # direction mode has S = 1, so KV[:, :ncols] is contiguous
            h.pf_reduced_hessian_batch(S, t["v"], t["theta"], t["lam"], t["y"], KV[:, :ncols],
                                       sigma_s=t["sigma_s"], sigma_x=t["sigma_x"], col0=col0, N=ncols, p_d=t["p_d"])
        K = allgather_columns(KV, n_u) if (directions and world > 1) else KV[:, :n_u]  # S = 1 when cpad > n_u
        if red_ev:
            red_ev[1].record(stream)
        if chol_ev:
            chol_ev[0].record(stream)
        reg["delta"], reg["trials"], reg["info"] = h.pf_condensed_kkt_solve_reg(S, K, t["sigma_u"], rhs=rhs, nrhs=1,
                                                                                 **REG)
        if chol_ev:
            chol_ev[1].record(stream)
        return KV

    if args.profile_steps:
        for _ in range(args.profile_steps):
            step(devt)
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        step(devt)
    torch.cuda.synchronize()
    # ------------------------------------------------------------ timed loop (device-resident inputs)
    launches0 = h.launch_count()
    step_ms, red_ms, chol_ms = [], [], []
    kern = {k: [] for k in h.KERNELS}
    deltas, trials = [], []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)  # outside the timed region
            e0, e1 = ev(), ev()
            re, ce = (ev(), ev()), (ev(), ev())
            e0.record(stream)
            step(devt, re, ce)
            e1.record(stream)
            torch.cuda.synchronize()
            step_ms.append(e0.elapsed_time(e1))
            red_ms.append(re[0].elapsed_time(re[1]))
            chol_ms.append(ce[0].elapsed_time(ce[1]))
            deltas.append(float(np.max(reg["delta"])))
            trials.append(int(np.max(reg["trials"])))
            assert not np.any(reg["info"]), "condensed KKT not positive definite within δ_max"
            for k, v in h.kernel_times().items():
                kern[k].append(v)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    launches = h.launch_count() - launches0
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, statistics.mean(red_ms), statistics.mean(chol_ms)], dtype=f64, device=dev)
    hv = torch.tensor([S * ncols], dtype=f64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(hv)
    total_ms, red_avg, chol_avg = t.tolist()
    hvps_per_step = hv.item()
    value = hvps_per_step * args.steps / (total_ms / 1e3)
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, {"rank": rank, "ms_per_step": sum(step_ms) / args.steps,
                                          "directions": S * ncols, "device": torch.cuda.get_device_name(dev)})
    else:
        per_rank = None

    # ------------------------------------------------------------ generic-HVP variant: dense V ~ N(0,1)
    generic = None
    if ncols > 0 and not args.no_generic:
        gen = torch.Generator(device=dev).manual_seed(7)
        Vd = torch.randn(S, ncols, n_u, generator=gen, dtype=f64, device=dev)
        gms = []
        h.pf_jacobian(S, devt["v"], devt["theta"])
        for k in range(args.warmup + args.steps):
            flush.fill_(1.0)
            e0, e1 = ev(), ev()
            e0.record(stream)
            h.pf_reduced_hessian_batch(S, devt["v"], devt["theta"], devt["lam"], devt["y"], KV[:, :ncols],
                                       sigma_s=devt["sigma_s"], sigma_x=devt["sigma_x"], V=Vd, N=ncols,
                                       p_d=devt["p_d"])
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                gms.append(e0.elapsed_time(e1))
        del Vd
        generic = {"value": S * ncols / (statistics.mean(gms) / 1e3), "unit": "HVP/s", "ms": statistics.mean(gms),
                   "directions": S * ncols, "V": "dense N(0,1), seed 7 (A7.1 a real SpMM)"}

    # ------------------------------------------------------------ the step's device work as one CUDA graph
    # (captured once, replayed: no host launch gaps); the condensed solve runs at the δ_w the loop
    # found (the loop's host decisions cannot be captured).  Context, not the headline.
    graph = None
    if ncols > 0 and (not directions or world == 1) and not args.no_graph:
        dmax = float(max(deltas))
        rhs_g = torch.empty(S, n_u, dtype=f64, device=dev)
        info_g = torch.empty(S, dtype=torch.int32, device=dev)
        h.profile(False)

        def gbody():
            rhs_g.copy_(devt["rhs"])
            h.pf_eval_constraints(S, devt["v"], devt["theta"], devt["p_g"], devt["q_g"], devt["p_d"], devt["q_d"], G, H)
            h.pf_jacobian(S, devt["v"], devt["theta"], info=info_j)
            h.pf_reduced_hessian_batch(S, devt["v"], devt["theta"], devt["lam"], devt["y"], KV[:, :ncols],
                                       sigma_s=devt["sigma_s"], sigma_x=devt["sigma_x"], N=ncols, p_d=devt["p_d"])
            h.pf_condensed_kkt_solve(S, KV[:, :n_u], devt["sigma_u"], dmax, rhs=rhs_g, nrhs=1, info=info_g)

        side = torch.cuda.Stream(dev)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            gbody()
        stream.wait_stream(side)
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            gbody()
        gms = []
        for k in range(args.warmup + args.steps):
            flush.fill_(1.0)
            e0, e1 = ev(), ev()
            e0.record(stream)
            cg.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                gms.append(e0.elapsed_time(e1))
        assert not torch.any(info_g != 0)
        graph = {"value": S * ncols / (statistics.mean(gms) / 1e3), "unit": "HVP/s", "ms_per_step": statistics.mean(gms),
                 "delta_w": dmax, "note": "eval + jacobian + reduction + condensed solve captured once as a CUDA "
                 "graph and replayed (L2 flushed between replays); the δ_w loop's host decisions are not captured"}
        del cg
        h.profile(True)

    # ------------------------------------------------------------ the NEXT rows' calls at the same point (ms per call, all S scenarios)
    next_rows = None
    if not args.no_next and rank == 0:
        L = h.kkt_len()
        r = torch.randn(S, L, generator=torch.Generator(device=dev).manual_seed(9), dtype=f64, device=dev)
        b = torch.empty(S, n_u, dtype=f64, device=dev)
        p = torch.empty(S, L, dtype=f64, device=dev)
        lam2, grad = torch.empty(S, n_x, dtype=f64, device=dev), torch.empty(S, n_u, dtype=f64, device=dev)
        h.pf_jacobian(S, devt["v"], devt["theta"])
        calls = {
            "pf_reduced_gradient (NEXT-2: adjoint λ + ∇f_r)": lambda: h.pf_reduced_gradient(
                S, devt["v"], devt["theta"], devt["p_g"], devt["y"], lam=lam2, grad=grad, p_d=devt["p_d"]),
            "pf_condensed_rhs (NEXT-1: Theorem 1/2 right-hand side)": lambda: h.pf_condensed_rhs(
                S, devt["v"], devt["theta"], devt["lam"], devt["y"], r, b=b, sigma_s=devt["sigma_s"],
                sigma_x=devt["sigma_x"], p_d=devt["p_d"]),
            "pf_recover_step (NEXT-1: p_x, p_s, p_λ, p_y)": lambda: h.pf_recover_step(
                S, devt["v"], devt["theta"], devt["lam"], devt["y"], r, b, p=p, sigma_s=devt["sigma_s"],
                sigma_x=devt["sigma_x"], p_d=devt["p_d"]),
        }
        next_rows = {}
        for name, fn in calls.items():
            ms = []
            for k in range(args.warmup + args.steps):
                e0, e1 = ev(), ev()
                e0.record(stream)
                fn()
                e1.record(stream)
                torch.cuda.synchronize()
                if k >= args.warmup:
                    ms.append(e0.elapsed_time(e1))
            next_rows[name] = {"ms": statistics.mean(ms), "scenarios": S}
        next_rows["pf_condensed_kkt_solve_reg (NEXT-3)"] = {"ms": chol_avg, "trials_max": max(trials),
                                                            "delta_w_max": max(deltas)}
        # NEXT-4: the LinRed IPM driver (Algorithm 1, host loop over the C-ABI) on case9 to 1e-8
        from paper_2203_11875_b200.ipm import LinRedIPM
        from synth import case9
        from synth.case9 import case9_bounds
        net9, pt9 = case9()
        b9, c0 = case9_bounds()
        solver = LinRedIPM(net9, b9, device=local, tol=1e-8)
        t0 = time.perf_counter()
        res = solver.solve(v0=pt9["v"], p_g0=pt9["p_g"])
        dt_ipm = time.perf_counter() - t0
        solver.close()
        next_rows["LinRed IPM (NEXT-4), case9 to 1e-8"] = {
            "status": res["status"], "iterations": res["iterations"], "objective_usd_per_h": res["objective"] + c0,
            "published_optimum_usd_per_h": 5296.69, "ms_per_iteration_wall": 1e3 * dt_ipm / max(1, res["iterations"])}

    # ------------------------------------------------------------ end-to-end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        pinned = {k: torch.from_numpy(a).pin_memory() for k, a in host.items()}
        out_rhs = torch.empty(S, n_u, dtype=f64).pin_memory()
        dt = {k: torch.empty_like(v) for k, v in devt.items()}
        h2d = sum(p_.numel() * p_.element_size() for p_ in pinned.values())
        d2h = out_rhs.numel() * 8
        e2e_ms = []
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.fill_(1.0)
            e0, e1 = ev(), ev()
            e0.record(stream)
            for k in dt:
                dt[k].copy_(pinned[k], non_blocking=True)
            step(dt)
            out_rhs.copy_(rhs, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        te = torch.tensor([sum(e2e_ms)], dtype=f64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": hvps_per_step * args.steps / (te.item() / 1e3), "unit": "HVP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h + 16 * S),
               "ms_per_step": te.item() / args.steps,
               "note": "host inputs copied in, the solution p_u and the δ_w loop's info/δ_w/trials copied out"}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ------------------------------------------------------------ rooflines
    peaks = read_peaks()
    hbm = peaks.get("hbm_gbs")
    dirs = S * ncols
    # algorithmic DRAM bytes per direction of each kernel: each slab row a
    # kernel must produce is written once and each row it must consume is read once
    # (gathers assumed cached); factors, network and line state are per-launch
    # constants (L2-resident) and are not counted.  The forward L sweep only visits
    # the tile's sparse-RHS reach (r rows), the Lᵀ sweep the ancestors of G_u's rows (a).
    ntc = -(-n_u // d["tile_cols"])
    r_mean = d["reach_rows_l"] / ntc if d["reach_rows_l"] else n_x
    a_rows = d["reach_rows_ua"] or n_x
    g_rows = d["gu_rows"] or n_x
    per_dir = {"k_fwd": 8.0 * (2 * r_mean + n_x),             # L sweep writes r rows; U reads them, writes Z
               "k_mu": 8.0 * 2 * n_g,                         # μ_A rows written (Z reads hit L2)
               "k_hvp": 8.0 * (2 * n_x + n_u),                # Z read, H_x write, H_u write
               "k_adj": 8.0 * (2 * n_x + 2 * a_rows),          # Uᵀ sweep r+w, Lᵀ sweep r+w on a rows
               "k_proj": 8.0 * (g_rows + 2 * n_u)}             # Ψ at G_u rows, H_u read, K̂V write
    kstats = {}
    for k, v in kern.items():
        v = [x for x in v if x >= 0]
        if not v:
            continue
        ms = statistics.mean(v)
        ach = per_dir[k] * dirs / (ms / 1e3) / 1e9 if per_dir.get(k) else None
        kstats[k] = {"ms": ms, "GBps": ach, "frac": (ach / hbm) if (ach and hbm) else None}
    dom = max((k for k in kstats if k in per_dir), key=lambda k: kstats[k]["ms"])
    traffic = {}
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(args.config, {})
    except Exception:
        pass
    # A9 on the FP64 pipe: S·n_u³/3 flops of the factorization (the solves are O(n_u²)) per launch
    chol_flops = S * n_u ** 3 / 3.0
    fp64 = None
    if "k_chol_dag" in kstats:
        tf = chol_flops / (kstats["k_chol_dag"]["ms"] / 1e3) / 1e12
        fp64 = {"bound": "fp64", "kernel": "k_chol_dag", "achieved": tf, "peak": FP64_PEAK_TFLOPS,
                "unit": "TFLOP/s", "frac": tf / FP64_PEAK_TFLOPS, "traffic": traffic.get("k_chol_dag"),
                "algorithmic_flops_per_launch": chol_flops, "kernel_ms": kstats["k_chol_dag"]["ms"],
                "peak_source": FP64_PEAK_SOURCE}
    lu = None
    if "k_lu" in kstats:
        sync_levels = max(1, d["front_level"] - d["lu_cut_level"])
        lu = {"kernel": "k_lu", "ms": kstats["k_lu"]["ms"], "levels": d["n_levels_l"],
              "us_per_level": 1e3 * kstats["k_lu"]["ms"] / d["n_levels_l"],
              "schedule": {"subtree_walk_levels": d["lu_cut_level"], "synchronised_levels": sync_levels,
                           "dense_front_rows": d["front_rows"], "front_level": d["front_level"]},
              "us_per_synchronised_level": 1e3 * kstats["k_lu"]["ms"] / sync_levels,
              "bound": "latency: each cluster-synchronised level waits for its longest row's IKJ chain "
                       "(staging + pivots); the bottom subtrees and the dense front are off that chain",
              "scenarios": S}
    roof = {"bound": "hbm", "achieved": kstats[dom]["GBps"], "peak": hbm, "unit": "GB/s",
            "frac": kstats[dom]["frac"], "traffic": traffic.get(dom), "kernel": dom,
            "algorithmic_bytes_per_direction": per_dir[dom], "directions_per_launch": dirs,
            "kernel_ms": kstats[dom]["ms"], "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
            "fp64_kernel": "k_chol_dag", "fp64_achieved_tflops": fp64 and fp64["achieved"],
            "fp64_peak_tflops": FP64_PEAK_TFLOPS, "fp64_frac": fp64 and fp64["frac"],
            "per_kernel": kstats}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # a bounded sample (~10 s of CPU work): whole scenarios of the same workload until 10 s have passed
        lam0 = oracle_lambda(net, pts[0])
        t0 = time.perf_counter()
        hv_cpu, nsc = 0, 0
        while nsc < len(pts) and (nsc == 0 or time.perf_counter() - t0 < 10.0):
            hv_cpu += oracle_step(net, pts[nsc], lam0 if nsc == 0 else oracle_lambda(net, pts[nsc]))[0]
            nsc += 1
        dtc = time.perf_counter() - t0
        cpu = {"value": hv_cpu / dtc, "unit": "HVP/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": "%d %s-shaped scenario(s), all %d directions each (naive-sensitivity oracle + the δ_w loop's "
                         "dense Cholesky), %.1f s" % (nsc, cfg["grid"], hv_cpu // max(nsc, 1), dtc)}

    line = {
        "metric": METRIC, "value": value, "unit": "HVP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if cfg["mode"] == "scenarios" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "%s (BASELINE.json configs[%d])" % (args.config, cfg["baseline_cfg"]),
                   "grid": cfg["grid"], "n_b": n_b, "n_l": n_l, "n_g": n_g, "n_x": n_x, "n_u": n_u, "m": m,
                   "scenarios_per_gpu": S, "directions_per_step": int(hvps_per_step),
                   "tile_cols": d["tile_cols"], "levels_l": d["n_levels_l"], "levels_u": d["n_levels_u"],
                   "nnz_lu": d["nnz_lu"], "lambda": "adjoint multipliers (pf_reduced_gradient), before timing",
                   "delta_w_max": max(deltas), "reg_trials_max": max(trials),
                   "parallelism": ("scenario-sharded x%d" % world) if cfg["mode"] == "scenarios"
                   else ("direction-sharded x%d + NCCL all-gather" % world),
                   "l2": "flushed between steps (256 MiB write outside the timed region)"},
        "chol_ms_per_iter": chol_avg, "reduction_ms_per_iter": red_avg,
        "reduction_ms_includes": "pf_jacobian (LU refactor) + pf_reduced_hessian_batch" +
                                 (" + NCCL all-gather" if directions and world > 1 else ""),
        "generic_hvp": generic, "cuda_graph": graph, "next_rows": next_rows,
        "roofline": roof, "roofline_fp64": fp64, "lu_latency": lu,
        "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(), "per_rank": per_rank,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
