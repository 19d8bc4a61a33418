#!/usr/bin/env python
"""bench.py — throughput of the batched reduced-Hessian hot path on B200.

One *step* = one IPM-iteration-equivalent of the whole hot path
over every scenario the rank owns:
  pf_eval_constraints (A2/A3) → pf_jacobian (A4 Jacobian values + A5 LU
  refactorization) → pf_reduced_hessian_batch over ALL n_u directions (A6,
  A7.1–A7.5) → [all-gather of column slabs, direction mode only] →
  pf_condensed_kkt_solve (A9: symmetrize + Σ_u + δ_w, FP64 Cholesky, solve).

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
import math
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
    ap.add_argument("--profile-steps", type=int, default=0, help="run N untimed steps and exit (for ncu)")
    ap.add_argument("--delta-w", type=float, default=None, help="skip the regularisation search (profiling)")
    ap.add_argument("--pipelines", type=int, default=1,
                    help="scenario groups run as independent handle+stream pipelines (scenario mode)")
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


def oracle_step(net, pt, delta_w):
    """The oracle (as it stands) for one scenario: Jacobians, K, the naive
    reduction, the condensed KKT Cholesky and solve.  Returns HVPs done."""
    import numpy as np
    from oracle import pf_oracle as O
    part = O.partition(net)
    O.constraints(net, pt)
    Gx, Gu, A = O.jacobians(net, part, pt)
    K = O.kkt_K(net, part, pt, pt["lam"], pt["y"], pt["sigma_s"], pt["sigma_x"])
    Kh = O.reduce_naive(K, Gx, Gu)
    Kc = O.condensed(0.5 * (Kh + Kh.T), pt["sigma_u"], delta_w)
    L, info = O.cholesky(Kc)
    if info == 0:
        O.chol_solve(L, np.ones(part["n_u"]))
    return part["n_u"]


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle on the box's host cores (rank 0 only)."""
    if rank != 0:
        return
    net, pts, _ = make_inputs(cfg, 0, 1)
    delta_w = 1e5
    for _ in range(args.warmup):
        oracle_step(net, pts[0], delta_w)
    t0 = time.perf_counter()
    hv = 0
    for k in range(args.steps):
        hv += oracle_step(net, pts[k % len(pts)], delta_w)
    dt = time.perf_counter() - t0
    value = hv / dt
    cores = cpu_threads()
    sample = "one %s-shaped scenario per step (all %d directions, naive-sensitivity oracle + dense Cholesky)" % (
        cfg["grid"], hv // args.steps)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "HVP/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak" if cfg["mode"] == "scenarios" else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "%s (BASELINE.json configs[%d])" % (args.config, cfg["baseline_cfg"]),
                       "grid": cfg["grid"], "n_b": net["n_b"], "n_l": net["n_l"], "n_g": net["n_g"],
                       "scenarios_per_gpu": cfg["scen"], "directions_per_step": hv // args.steps,
                       "parallelism": "CPU oracle, rank 0 only"},
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
    # P independent pipelines (one handle + one stream each) over contiguous scenario
    # groups: the latency-bound phases of one group (LU refactor, Cholesky chain)
    # overlap the bandwidth-bound reduction of the other.
    P = args.pipelines if (not directions and S % max(args.pipelines, 1) == 0) else 1
    Sg = S // P
    hs = [Network(net, max_batch=max(cpad, 1), max_scen=Sg, device=local, tile_cols=tile if directions else 0)
          for _ in range(P)]
    h = hs[0]
    h.profile(True)
    d = h.dims

    def stack(key):
        return np.ascontiguousarray(np.stack([np.asarray(p[key], dtype=np.float64) for p in pts]))

    host = {k: stack(k) for k in ("v", "theta", "p_g", "q_g", "p_d", "q_d", "lam", "y", "sigma_s", "sigma_x",
                                  "sigma_u")}
    host["rhs"] = np.ones((S, n_u))
    devt = {k: torch.as_tensor(a, device=dev) for k, a in host.items()}
    G = torch.empty(S, 2 * n_b, dtype=f64, device=dev)
    H = torch.empty(S, 2 * n_l, dtype=f64, device=dev)
    info_j = torch.empty(S, dtype=torch.int32, device=dev)
    info_c = torch.empty(S, dtype=torch.int32, device=dev)
    KV = torch.empty(S, cpad, n_u, dtype=f64, device=dev)
    rhs = torch.empty(S, n_u, dtype=f64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    streams = [stream] if P == 1 else [torch.cuda.Stream(dev) for _ in range(P)]
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def step(t, red_ev=None, chol_ev=None):
        go = torch.cuda.Event()
        go.record(stream)
        rhs.copy_(t["rhs"])
        done = []
        for g, (hg, sg) in enumerate(zip(hs, streams)):
            a, b = g * Sg, (g + 1) * Sg
            sl = {k: v[a:b] for k, v in t.items()}
            sg.wait_event(go)
            if sg is not stream:
                sg.wait_stream(stream)
            with torch.cuda.stream(sg):
                hg.pf_eval_constraints(Sg, sl["v"], sl["theta"], sl["p_g"], sl["q_g"], sl["p_d"], sl["q_d"],
                                       G[a:b], H[a:b])
                hg.pf_jacobian(Sg, sl["v"], sl["theta"], info=info_j[a:b])
                if red_ev and g == 0:
                    red_ev[0].record(sg)
                if ncols > 0:  # direction mode has S = 1, so KV[:, :ncols] is contiguous
                    hg.pf_reduced_hessian_batch(Sg, sl["v"], sl["theta"], sl["lam"], sl["y"], KV[a:b, :ncols],
                                                sigma_s=sl["sigma_s"], sigma_x=sl["sigma_x"], col0=col0, N=ncols,
                                                p_d=sl["p_d"])
                if red_ev and g == 0:
                    red_ev[1].record(sg)
                K = allgather_columns(KV, n_u) if (directions and world > 1) else KV[a:b]
                if chol_ev and g == 0:
                    chol_ev[0].record(sg)
                hg.pf_condensed_kkt_solve(Sg, K, sl["sigma_u"], delta_w, rhs[a:b], 1, info_c[a:b])
                if chol_ev and g == 0:
                    chol_ev[1].record(sg)
            if sg is not stream:
                e = torch.cuda.Event()
                e.record(sg)
                done.append(e)
        for e in done:
            stream.wait_event(e)
        return KV

    # ------------------------------------------------------------ δ_w: the paper's regularisation until PD
    delta_w = 0.0 if args.delta_w is None else args.delta_w
    for k in ([None] + list(range(-8, 12))) if args.delta_w is None else []:
        delta_w = 0.0 if k is None else 10.0 ** k
        step(devt)
        torch.cuda.synchronize()
        ok = torch.zeros(1, device=dev) + (info_c != 0).sum()
        if world > 1:
            dist.all_reduce(ok)
        if ok.item() == 0:
            break
    if args.profile_steps:
        for _ in range(args.profile_steps):
            step(devt)
        torch.cuda.synchronize()
        return

    for _ in range(args.warmup):
        step(devt)
    torch.cuda.synchronize()
    # ------------------------------------------------------------ timed loop (device-resident inputs)
    launches0 = sum(x.launch_count() for x in hs)
    step_ms, red_ms, chol_ms = [], [], []
    kern = {k: [] for k in h.KERNELS}
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
            for k, v in h.kernel_times().items():
                kern[k].append(v)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    launches = sum(x.launch_count() for x in hs) - launches0
    total_ms = sum(step_ms)
    t = torch.tensor([total_ms, statistics.mean(red_ms), statistics.mean(chol_ms)], dtype=f64, device=dev)
    hv = torch.tensor([S * ncols], dtype=f64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.all_reduce(hv)
    total_ms, red_avg, chol_avg = t.tolist()
    hvps_per_step = hv.item()
    value = hvps_per_step * args.steps / (total_ms / 1e3)

    # ------------------------------------------------------------ generic-HVP variant: dense V ~ N(0,1)
    generic = None
    if ncols > 0 and not args.no_generic:
        gen = torch.Generator(device=dev).manual_seed(7)
        Vd = torch.randn(Sg, ncols, n_u, generator=gen, dtype=f64, device=dev)
        gms = []
        for k in range(args.warmup + args.steps):
            flush.fill_(1.0)
            e0, e1 = ev(), ev()
            e0.record(stream)
            h.pf_reduced_hessian_batch(Sg, devt["v"][:Sg], devt["theta"][:Sg], devt["lam"][:Sg], devt["y"][:Sg],
                                       KV[:Sg, :ncols], sigma_s=devt["sigma_s"][:Sg], sigma_x=devt["sigma_x"][:Sg],
                                       V=Vd, N=ncols, p_d=devt["p_d"][:Sg])
            e1.record(stream)
            torch.cuda.synchronize()
            if k >= args.warmup:
                gms.append(e0.elapsed_time(e1))
        del Vd
        generic = {"value": Sg * ncols / (statistics.mean(gms) / 1e3), "unit": "HVP/s", "ms": statistics.mean(gms),
                   "directions": Sg * ncols, "V": "dense N(0,1), seed 7 (A7.1 a real SpMM)"}

    # ------------------------------------------------------------ end-to-end through the public API, host buffers
    e2e = None
    if not args.no_e2e:
        pinned = {k: torch.from_numpy(a).pin_memory() for k, a in host.items()}
        out_rhs = torch.empty(S, n_u, dtype=f64).pin_memory()
        out_info = torch.empty(S, dtype=torch.int32).pin_memory()
        dt = {k: torch.empty_like(v) for k, v in devt.items()}
        h2d = sum(p.numel() * p.element_size() for p in pinned.values())
        d2h = out_rhs.numel() * 8 + out_info.numel() * 4
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
            out_info.copy_(info_c, non_blocking=True)
            e1.record(stream)
            torch.cuda.synchronize()
            e2e_ms.append(e0.elapsed_time(e1))
        te = torch.tensor([sum(e2e_ms)], dtype=f64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e = {"value": hvps_per_step * args.steps / (te.item() / 1e3), "unit": "HVP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": te.item() / args.steps}

    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ------------------------------------------------------------ roofline of the dominant kernel
    peaks = read_peaks()
    hbm = peaks.get("hbm_gbs")
    dirs = Sg * ncols  # per launch: the kernels of pipeline 0 (its Sg scenarios)
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
               "k_proj": 8.0 * (g_rows + 2 * n_u),             # Ψ at G_u rows, H_u read, K̂V write
               "k_lu": None}
    kstats = {}
    for k, v in kern.items():
        if not v:
            continue
        ms = statistics.mean(v)
        ach = per_dir[k] * dirs / (ms / 1e3) / 1e9 if per_dir.get(k) else None
        kstats[k] = {"ms": ms, "GBps": ach, "frac": (ach / hbm) if (ach and hbm) else None}
    dom = max((k for k in kstats if k != "k_lu"), key=lambda k: kstats[k]["ms"])
    traffic = None
    try:
        tj = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
        traffic = tj.get(args.config, {}).get(dom)
    except Exception:
        pass
    roof = {"bound": "hbm", "achieved": kstats[dom]["GBps"], "peak": hbm, "unit": "GB/s",
            "frac": kstats[dom]["frac"], "traffic": traffic, "kernel": dom,
            "algorithmic_bytes_per_direction": per_dir[dom], "directions_per_launch": dirs,
            "kernel_ms": kstats[dom]["ms"], "peak_source": "MEASURED_PEAKS.json hbm_gbs (measured)",
            "per_kernel": kstats}

    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # a bounded sample (~10 s of CPU work): whole scenarios of the same workload until 10 s have passed
        t0 = time.perf_counter()
        hv_cpu, nsc = 0, 0
        while nsc < len(pts) and (nsc == 0 or time.perf_counter() - t0 < 10.0):
            hv_cpu += oracle_step(net, pts[nsc], delta_w)
            nsc += 1
        dtc = time.perf_counter() - t0
        cpu = {"value": hv_cpu / dtc, "unit": "HVP/s", "cores": cpu_threads(), "kind": "oracle",
               "sample": "%d %s-shaped scenario(s), all %d directions each (naive-sensitivity oracle + dense Cholesky), "
                         "%.1f s" % (nsc, cfg["grid"], hv_cpu // max(nsc, 1), dtc)}

    line = {
        "metric": METRIC, "value": value, "unit": "HVP/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if cfg["mode"] == "scenarios" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "%s (BASELINE.json configs[%d])" % (args.config, cfg["baseline_cfg"]),
                   "grid": cfg["grid"], "n_b": n_b, "n_l": n_l, "n_g": n_g, "n_x": n_x, "n_u": n_u, "m": m,
                   "scenarios_per_gpu": S, "directions_per_step": int(hvps_per_step),
                   "tile_cols": d["tile_cols"], "levels_l": d["n_levels_l"], "levels_u": d["n_levels_u"],
                   "nnz_lu": d["nnz_lu"], "delta_w": delta_w,
                   "pipelines_per_gpu": P,
                   "parallelism": ("scenario-sharded x%d" % world) if cfg["mode"] == "scenarios"
                   else ("direction-sharded x%d + NCCL all-gather" % world),
                   "l2": "flushed between steps (256 MiB write outside the timed region)"},
        "chol_ms_per_iter": chol_avg, "reduction_ms_per_iter": red_avg,
        "generic_hvp": generic,
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
