#!/usr/bin/env python
"""Benchmark of the B200 PFE solver (BASELINE.json metric: PFE inner
iterations/s and PCG SpMV HBM GB/s as a fraction of peak).

One *step* = one full PFE solve (soc: soc_max outer x sb_max inner
iterations) of the configured workload, from Y0 already resident in HBM.
Default workload: BASELINE.json configs[1] (C2, 481x321 Voronoi image,
8-neighbour grid, d=4, 10x20, Jacobi-PCG tol 1e-6).

Arms:
  (default)         sm_100a library; value = inner iterations / s over K timed
                    steps (CUDA events, L2 flushed between steps); e2e = the same
                    metric through the one-call C ABI ``pfe_solve`` with host
                    buffers (graph + Y0 in, Y out) per step.
  --impl reference  the reference's CPU implementation of the path.  The
                    reference needs Eigen3 (absent), so this times the oracle
                    port (oracle/, an Eigen-free C++ restatement) on all host
                    threads it can use (one per embedding column); each step is
                    a bounded sample (first outer iteration = sb_max inner
                    iterations).

Multi-GPU (torchrun, N>1): every rank solves its own independent image of the
same configuration (different seed: a dataset of images, weak scaling, no
collective on the data path); value = total inner iterations / max-over-ranks
time.
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
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "PFE inner iters/sec (PCG SpMV HBM GB/s fraction reported in roofline)"
UNIT = "inner_iters/s"


# ----------------------------------------------------------------- helpers --
def dist_init(n_gpus):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce_max(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def allreduce_sum(x, world):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(config, kernel):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        return json.loads(p.read_text()).get(config, {}).get(kernel)
    except Exception:
        return None


def algorithmic_bytes(kind, n, m, d):
    """Contract bytes per launch."""
    nd = n * d
    if kind == "pcg_spmv":      # read r, p_old; write p, q; edge weights, diag, inv_diag
        return 32 * nd + 8 * m + 16 * n
    if kind == "pcg_update":    # read x, p, q, r; write x, r; inv_diag
        return 48 * nd + 8 * n
    if kind == "pcg_init":      # read x0, rhs; write r, p; operator
        return 32 * nd + 8 * m + 16 * n
    if kind == "sb_pass":       # read Y, b, w, rq; write b, rhs
        return 16 * m * d + 24 * nd + 8 * m
    return None


# ------------------------------------------------------------------ arms ---
def sample_inner(cfg, core_seconds):
    """Inner iterations of the oracle that fit in ~core_seconds of single-core
    work: C2's 20 inner iterations take ~1.8 s, and the cost scales with the
    (m + n) d of the graph."""
    d = cfg.params.dim
    est = 0.09 * (cfg.graph.m * d + cfg.graph.n * d) / (613454 * 4 + 154401 * 4)
    return int(max(1, min(cfg.params.sb_max_stage1, core_seconds // max(est, 1e-9))))


def run_reference(args, rank, world):
    if rank != 0:
        return None
    from paper_1612_06496_b200.inputs import make_config
    from paper_1612_06496_b200 import api

    sys.path.insert(0, str(ROOT / "tests"))
    import oracle as O

    cfg = make_config(args.config, seed=0)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    threads = min(prm.dim, os.cpu_count() or 1)
    O.set_threads(threads)
    sample = api.PfeParams(**{**prm.__dict__})
    sample.soc_max = 1
    sample.sb_max_stage1 = sample_inner(cfg, 10.0 * threads)  # <= ~10 s per step on `threads` cores
    inner = sample.sb_max_stage1
    for _ in range(args.warmup if args.warmup < 1 else 1):
        O.solve(g, sample, y0, mode=0)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.solve(g, sample, y0, mode=0)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    val = args.steps * inner / tot
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Voronoi image, BASELINE.json configs[1] shape)",
            "config": {"workload": cfg.name, "description": cfg.description, "n": g.n, "m": g.m, "d": prm.dim,
                       "inner_per_step": inner},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"first outer iteration ({inner} inner iterations) of {cfg.name}, "
                                       f"oracle port (reference needs Eigen3, absent), {threads} column threads "
                                       f"of {os.cpu_count()} host cores"},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    return line


def cpu_baseline(cfg, y0):
    """Oracle port on 1 host core, bounded sample: one outer iteration."""
    from paper_1612_06496_b200 import api

    sys.path.insert(0, str(ROOT / "tests"))
    import oracle as O

    O.set_threads(1)
    sample = api.PfeParams(**{**cfg.params.__dict__})
    sample.soc_max = 1
    sample.sb_max_stage1 = sample_inner(cfg, 15.0)
    t0 = time.perf_counter()
    O.solve(cfg.graph, sample, y0, mode=0)
    dt = time.perf_counter() - t0
    inner = sample.sb_max_stage1
    return {"value": inner / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"first outer iteration truncated to {inner} inner iterations ({dt:.1f} s incl. operator "
                      f"set-up and one projection) of {cfg.name} on 1 of {os.cpu_count()} host cores; oracle "
                      f"port (reference needs Eigen3, absent)"}


def run_bands(args, rank, world, local):
    """Strong scaling of ONE image split into row bands, one band per GPU (NCCL halos)."""
    import torch
    import torch.distributed as dist

    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import make_config

    cfg = make_config(args.config, seed=0)  # the same image on every rank
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    inner_per_step = prm.soc_max * prm.sb_max_stage1
    obj = [api.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    torch.cuda.set_device(local)
    solver = api.BandSolver(g, prm, obj[0], world, rank, device=local, warn=False)
    st = solver.make_state(y0)
    for _ in range(args.warmup):
        st.reset()
        solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    barrier(world)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            st.reset()
            barrier(world)
            solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)
            times.append(solver.last_ms() * 1e-3)
    t_max = allreduce_max(sum(times), world)
    # end to end: state from host y0, solve, gathered Y back on the host
    e2e = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s2 = solver.make_state(y0)
        solver.run_soc(s2, prm.soc_max, prm.sb_max_stage1)
        _ = s2.y
        e2e.append(time.perf_counter() - t0)
        s2.close()
    e2e_max = allreduce_max(sum(e2e), world)
    if rank != 0:
        return None
    rep = solver.report()
    return {
        "metric": METRIC, "value": args.steps * inner_per_step / t_max, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded Voronoi RGB image)",
        "config": {"workload": cfg.name, "description": cfg.description, "n": g.n, "m": g.m, "d": prm.dim,
                   "parallelism": (f"{world} row bands (NCCL halo exchange + gathered PCG totals)" if g.grid else f"{world} vertex ranges (NCCL ghost-row exchange + gathered PCG totals)"),
                   "l2": "inputs larger than L2" if g.n * prm.dim * 8 > 126e6 else "resident",
                   "topology": ["csr", "grid8", "grid24"][rep["topology"]]},
        "roofline": None,
        "cpu_baseline": None,
        "e2e": {"value": args.steps * inner_per_step / e2e_max, "unit": UNIT,
                "h2d_bytes_per_step": g.n * prm.dim * 8, "d2h_bytes_per_step": g.n * prm.dim * 8,
                "call": "BandSolver.make_state(y0) + run_soc + gathered state.y"},
        "gpu_launches": None,
        "clocks": clk.summary(),
    }


def run_gpu(args, rank, world, local):
    import ctypes as C

    from paper_1612_06496_b200 import _native as N
    from paper_1612_06496_b200 import api
    from paper_1612_06496_b200.inputs import make_config

    dev = local if world > 1 else args.device
    cfg = make_config(args.config, seed=rank)
    g, prm = cfg.graph, cfg.params
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    inner_per_step = prm.soc_max * prm.sb_max_stage1

    # ---- device-resident timing (value)
    solver = api.PfeSolver(g, prm, device=dev, use_graphs=not args.host_driven, warn=False,
                           persistent=not args.no_persistent)
    st = solver.make_state(y0)
    import torch

    torch.cuda.set_device(dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{dev}")
    for _ in range(args.warmup):
        st.reset()
        solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    torch.cuda.synchronize()
    barrier(world)
    ev = []
    with ClockSampler(dev) as clk:
        torch.cuda.synchronize()
        for _ in range(args.steps):
            flush.add_(1.0)  # evict L2 between steps (256 MB > 126 MB L2)
            st.reset()
            torch.cuda.synchronize()
            solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)  # synchronizes at the end
            ev.append(solver.last_ms() * 1e-3)  # CUDA events on the solver stream
        torch.cuda.synchronize()
    barrier(world)
    local_t = sum(ev)
    t_max = allreduce_max(local_t, world)
    rep = solver.report()
    its, _, _ = solver.pcg_log()
    last = its[-inner_per_step:]
    k_per_inner = last.max(axis=1)
    if rep["topology"] != 0 and not args.no_persistent:
        launches_per_step = 4 * prm.soc_max + 1  # persistent kernel + 3 projection kernels per outer, rhs_quad
    else:
        launches_per_step = int((2 * k_per_inner + 4).sum() + 3 * prm.soc_max + 1)
    total_inner = allreduce_sum(args.steps * inner_per_step, world)
    value = total_inner / t_max

    # ---- roofline of the dominant kernel: one instrumented step after the
    # timed region with CUDA events around every launch on the solver stream
    peak, peak_src = measured_peak()

    def instrumented(persistent):
        s = api.PfeSolver(g, prm, device=dev, use_graphs=False, warn=False, profile=True, persistent=persistent)
        ps = s.make_state(y0)
        s.run_soc(ps, prm.soc_max, prm.sb_max_stage1)  # warm (attributes, occupancy)
        s.kernel_times(reset=True)
        flush.add_(1.0)
        torch.cuda.synchronize()
        ps.reset()
        before = s.report()["inner_iterations"]
        s.run_soc(ps, prm.soc_max, prm.sb_max_stage1)
        kt = s.kernel_times()
        its, _, _ = s.pcg_log()
        k_inner = its[before:].max(axis=1)
        kind = s.report()["persistent_kind"]
        s.close()
        return kt, k_inner, kind

    # multi-kernel path: per-kernel split (also the path k-NN graphs use)
    kt_m, _, _ = instrumented(False)
    share = {k: v[0] for k, v in kt_m.items()}
    tot_ms = sum(share.values()) or 1.0
    per_kernel = {}
    for k in ("pcg_spmv", "pcg_update", "pcg_init", "sb_pass"):
        ms, cnt = kt_m[k]
        b = algorithmic_bytes(k, g.n, g.m, prm.dim)
        if cnt and b:
            gbs = b / (ms / cnt * 1e-3) / 1e9
            per_kernel[k] = {"avg_us": 1e3 * ms / cnt, "launches": cnt, "alg_bytes": b, "GB/s": gbs,
                             "frac": gbs / peak, "share": share[k] / tot_ms}
    persistent_used = rep["topology"] != 0 and not args.no_persistent
    if persistent_used:
        # the persistent kernel runs whole split_bregman calls: its algorithmic
        # bytes are those of every phase it executes
        bi = algorithmic_bytes("pcg_init", g.n, g.m, prm.dim)
        bs = algorithmic_bytes("pcg_spmv", g.n, g.m, prm.dim)
        bu = algorithmic_bytes("pcg_update", g.n, g.m, prm.dim)
        bsb = algorithmic_bytes("sb_pass", g.n, g.m, prm.dim)

        def persistent_roofline(mode):
            kt_p, k_inner, kind = instrumented(mode)
            ms, cnt = kt_p["sb_persistent"]
            total_b = float(sum(bi + int(k) * (bs + bu) + bsb for k in k_inner))
            return kind, ms, cnt, total_b, total_b / (ms * 1e-3) / 1e9

        kind, ms, cnt, total_b, gbs = persistent_roofline(True)
        kname = {1: "k_sb_persistent", 2: "k_sb_resident"}.get(kind, "k_sb_persistent")
        tiled = None
        if kind == 2:  # the streaming (tiled) persistent kernel on the same workload, for comparison
            _, ms_t, cnt_t, tb_t, gbs_t = persistent_roofline("tiled")
            tiled = {"kernel": "k_sb_persistent", "avg_launch_us": 1e3 * ms_t / cnt_t, "GB/s": gbs_t,
                     "frac": gbs_t / peak}
        roofline = {"bound": "hbm", "kernel": kname, "achieved": gbs, "peak": peak, "unit": "GB/s",
                    "frac": gbs / peak, "traffic": ncu_traffic(cfg.name, kname),
                    "peak_source": peak_src, "alg_bytes_per_launch": total_b / cnt,
                    "avg_launch_us": 1e3 * ms / cnt, "launches": cnt,
                    "model": ("compulsory bytes of the streamed algorithm (every PCG / split-Bregman phase "
                              "reads and writes its operands once, DESIGN.md §4) / kernel time"
                              + ("; k_sb_resident keeps the PCG state in shared memory, so its real HBM "
                                 "traffic is far below this and frac > 1 is possible: it is bounded by grid "
                                 "barrier latency, see profiles/" if kind == 2 else "")),
                    "timing": "CUDA events around every launch of one instrumented step after the timed region",
                    "tiled_persistent": tiled,
                    "kernels_multi_kernel_path": per_kernel}
    else:
        dom = max(("pcg_spmv", "pcg_update", "sb_pass"), key=lambda k: share[k])
        dk = per_kernel[dom]
        roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["GB/s"], "peak": peak, "unit": "GB/s",
                    "frac": dk["GB/s"] / peak, "traffic": ncu_traffic(cfg.name, dom), "peak_source": peak_src,
                    "alg_bytes_per_launch": dk["alg_bytes"], "avg_launch_us": dk["avg_us"],
                    "timing": "CUDA events around every launch of one instrumented step after the timed region",
                    "kernels": per_kernel}

    # ---- end to end through the one-call C ABI with host buffers
    gc, pc = g.to_c(), prm.to_c()
    xc = N.pfe_exec(dev, 1, 0, 0, 0 if args.no_persistent else 1)
    y0c = np.asfortranarray(y0)
    yout = np.empty(g.n * prm.dim)
    repc = N.pfe_report()
    lib = N.load()
    e2e_t = []
    for i in range(args.e2e_warmup + args.steps):
        t0 = time.perf_counter()
        rc = lib.pfe_solve(C.byref(gc), C.byref(pc), C.byref(xc), 0, N.dptr(y0c), N.dptr(yout), C.byref(repc))
        dt = time.perf_counter() - t0
        if rc != 0:
            raise RuntimeError(lib.pfe_last_error().decode())
        if i >= args.e2e_warmup:
            e2e_t.append(dt)
    e2e_max = allreduce_max(sum(e2e_t), world)
    h2d = g.m * (4 + 4 + 8) + g.n * 8 + g.n * prm.dim * 8
    d2h = g.n * prm.dim * 8

    result = None
    if rank == 0:
        cpu = cpu_baseline(cfg, y0) if (world == 1 and not args.no_cpu_baseline) else None
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Voronoi RGB image standing in for BSDS500; BASELINE.json configs[1] shape)",
            "config": {"workload": cfg.name, "description": cfg.description, "n": g.n, "m": g.m, "d": prm.dim,
                       "outer": prm.soc_max, "inner": prm.sb_max_stage1, "pcg_tol": prm.pcg.rel_tol,
                       "pcg_max_iter": prm.pcg.max_iter, "lambda": prm.lambda_, "r": prm.r,
                       "precond": "jacobi", "l2": "flushed between steps (256 MB write)",
                       "parallelism": f"{world} independent replicas" if world > 1 else "single GPU",
                       "pcg_iters_per_inner_mean": float(k_per_inner.mean()),
                       "topology": ["csr", "grid8", "grid24"][rep["topology"]],
                       "mode": ("persistent cooperative kernel per split_bregman call"
                                if rep["topology"] != 0 and not args.no_persistent else
                                ("host-driven" if args.host_driven else "cuda-graph (device WHILE loop)"))},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": {"value": total_inner / e2e_max, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "call": "pfe_solve (solver create + state + soc + download), host buffers"},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
        }
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c2")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--host-driven", action="store_true")
    ap.add_argument("--no-persistent", action="store_true", help="one kernel per phase instead of the "
                    "persistent cooperative kernel (grid graphs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--bands", action="store_true", help="N>1: split one image of a grid config into row "
                    "bands, one per GPU (strong scaling) instead of independent replicas")
    args = ap.parse_args()
    rank, world, local = dist_init(args.gpus)
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    elif args.bands and world > 1:
        line = run_bands(args, rank, world, local)
    else:
        line = run_gpu(args, rank, world, local)
    if rank == 0 and line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
