#!/usr/bin/env python
"""Benchmark of the B200 PFE solver (BASELINE.json metric: PFE inner
iterations/s and PCG SpMV HBM GB/s as a fraction of peak).

One *step* = one full PFE solve (soc: soc_max outer x sb_max inner
iterations) of the configured workload, from Y0 already resident in HBM.
Default workload: BASELINE.json configs[3] = C4 (4096x4096 Voronoi image,
8-neighbour grid, n = 16.8 M, d = 8, 5 x 20, Jacobi-PCG tol 1e-6): the
largest configuration that fits one GPU, whose state (Y, b, s: ~10 GB) streams
from HBM on every inner iteration, and north_star's scaling configuration.
``--config c1..c5`` selects another one.

Arms:
  (default)         sm_100a library; value = inner iterations / s over K timed
                    steps (CUDA events on the solver stream, L2 flushed between
                    steps); e2e = the same metric through the one-call C ABI
                    ``pfe_solve`` with host buffers (graph + Y0 in, Y out).
  --impl reference  the reference's CPU implementation of the path.  The
                    reference needs Eigen3 (absent), so this times the oracle
                    port (oracle/, the Eigen-free C++ restatement) on all host
                    threads it can use (one per embedding column, elementwise
                    loops split across all cores).  The solver is built once
                    (set-up reported, not timed); each step runs the next
                    inner iteration(s) of the same soc schedule and only the
                    inner iterations are timed.  No libpfe_b200.so is loaded.

Multi-GPU (torchrun, N>1): C3 / C4 split ONE image into N row bands and C5
splits its vertices into N ranges (NCCL halo / ghost-row exchange, gathered
PCG totals; strong scaling); C1 / C2 (single-GPU configurations) run N
independent replicas.  value = total inner iterations / max-over-ranks time.
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
SHARDED = ("c3", "c4", "c5")  # configurations BASELINE.json scales over GPUs


# ----------------------------------------------------------------- helpers --
def dist_init():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("gloo")  # host-side timing / control only; the data path uses NCCL
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def allreduce(x, world, op="max"):
    if world <= 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
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
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of a
    kernel on a workload, from this round's committed ncu --set full capture."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        row = json.loads(p.read_text()).get(config, {})
        return row.get(kernel, row.get(kernel[2:] if kernel.startswith("k_") else kernel))
    except Exception:
        return None


def algorithmic_bytes(topology, n, m, d):
    """Contract bytes per launch, SURVEY.md §8(d) (every array counted once).

    O_A (operator bytes): grid 8(m + n) (one weight per undirected edge + A_ii,
    stencil indices implicit); k-NN / CSR 24m + 12n + 4 (int32 column + fp64
    value per directed entry, row_ptr, A_ii)."""
    nd = n * d
    csr = topology == "csr"
    o_a = 24 * m + 12 * n + 4 if csr else 8 * (m + n)
    spmv = 32 * nd + o_a                 # p' = D^-1 r + beta p fused with q = A p', p'.q
    update = 48 * nd + 8 * n             # x += a p, r -= a q, r.r, r.D^-1 r
    init = 32 * nd + o_a                 # r = b - A x0, p = D^-1 r, norms
    sb = 16 * m * d + 24 * nd + 8 * m + ((4 * m + 4 * n) if csr else 0)  # shrink / Bregman / next rhs
    return {"pcg_spmv": spmv, "pcg_update": update, "pcg_init": init, "sb_pass": sb,
            "pcg_iteration": spmv + update, "outer": 72 * nd + 24 * n, "o_a": o_a}


def inner_bytes(b, k_per_inner):
    """Sum over inner iterations j of B_sb + B_init + k_j B_it."""
    return float(sum(b["sb_pass"] + b["pcg_init"] + int(k) * b["pcg_iteration"] for k in k_per_inner))


def load_config(name, seed=0):
    """The seeded synthetic workload.  C5's 16-NN graph is built on the GPU by
    pfe_knn_graph; for the CPU reference arm that build runs in a child
    process so the reference process never maps libpfe_b200.so."""
    from paper_1612_06496_b200.inputs import make_config

    return make_config(name, seed=seed)


def load_config_cpu_only(name, seed=0):
    if name != "c5":
        return load_config(name, seed)
    from paper_1612_06496_b200 import inputs

    cache = Path(os.environ.get("TMPDIR", "/tmp")) / f"pfe_bench_{name}_{seed}.npz"
    if not cache.exists():
        code = ("import sys,numpy as np; sys.path.insert(0, %r); from paper_1612_06496_b200.inputs import make_config;"
                "c = make_config(%r, seed=%d); g = c.graph;"
                "np.savez(%r, n=g.n, ei=g.ei, ej=g.ej, w=g.w, degree=g.degree, sigma=g.sigma)"
                % (str(ROOT), name, seed, str(cache)))
        subprocess.run([sys.executable, "-c", code], check=True)
    z = np.load(cache)
    real = inputs.knn_graph
    try:  # make_config(c5) with its GPU graph build replaced by the cached result
        inputs.knn_graph = lambda pts, k, gpu=False: inputs.WeightedGraph(int(z["n"]), z["ei"], z["ej"], z["w"],
                                                                          z["degree"], float(z["sigma"]))
        return inputs.make_config(name, seed=seed)
    finally:
        inputs.knn_graph = real


def workload(cfg, topology):
    """The `config` object of both arms (same workload, same keys)."""
    g, prm = cfg.graph, cfg.params
    return {"workload": cfg.name, "description": cfg.description, "n": g.n, "m": g.m, "d": prm.dim,
            "outer": prm.soc_max, "inner": prm.sb_max_stage1, "pcg_tol": prm.pcg.rel_tol,
            "pcg_max_iter": prm.pcg.max_iter, "lambda": prm.lambda_, "r": prm.r, "precond": "jacobi",
            "topology": topology, "y0": f"random_embedding(n, d, seed={cfg.y0_seed}, degree)",
            "l2": "flushed between steps (256 MB write); the working set (Y, b, s) exceeds the 126 MB L2"
            if g.m * prm.dim * 8 > 126e6 else "flushed between steps (256 MB write)"}


def topology_of(cfg):
    g = cfg.graph
    if not g.grid:
        return "csr"
    return {1: "grid8", 2: "grid24"}[g.grid[2]]


DATA = ("synthetic (seeded Voronoi RGB images standing in for BSDS500 / seeded Gaussian-mixture point sets, "
        "BASELINE.json config shapes; inputs.py)")


# ------------------------------------------------------------ CPU legs ---
class pinned_to_core0:
    """Pins the calling thread (and threads it starts) to host core 0."""

    def __enter__(self):
        self.prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {sorted(self.prev)[0]})
        return sorted(self.prev)[0]

    def __exit__(self, *a):
        os.sched_setaffinity(0, self.prev)


def cpu_baseline(cfg, budget_s=20.0):
    """The oracle port on ONE pinned host core: a resident oracle solve of
    the same workload, the first inner iterations of its soc schedule
    timed (set-up and projections excluded, reported separately)."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle as O

    g, prm = cfg.graph, cfg.params
    y0 = O.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    O.set_threads(1)
    with pinned_to_core0() as core:
        sess = O.Session(g, prm, y0)
        t_in, t_out, ks = 0.0, 0.0, []
        while True:
            ti, to, k = sess.step(1)
            t_in += ti
            t_out += to
            ks.extend(int(v) for v in k)
            if t_in >= budget_s or len(ks) >= prm.soc_max * prm.sb_max_stage1:
                break
        sess.close()
    inner = len(ks)
    return {"value": inner / t_in, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": (f"first {inner} inner iteration(s) of the {cfg.name} soc schedule, {t_in:.1f} s of inner-loop "
                       f"time on host core {core} (taskset-style affinity, 1 of {os.cpu_count()} cores); oracle port "
                       f"(the reference needs Eigen3, absent); operator set-up {sess.setup_s:.1f} s and projections "
                       f"{t_out:.2f} s not timed"),
            "setup_s": sess.setup_s, "pcg_iters_per_inner": float(np.mean(ks))}


def run_reference(args, rank, world):
    """--impl reference: the oracle port of the reference's CPU solver on all
    host threads, same config / metric; rank 0 only."""
    if rank != 0:
        return None
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle as O

    cfg = load_config_cpu_only(args.config)
    g, prm = cfg.graph, cfg.params
    y0 = O.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)  # == pfe_random_embedding, bitwise
    threads = os.cpu_count() or 1
    O.set_threads(threads)
    sess = O.Session(g, prm, y0)
    total_inner = prm.soc_max * prm.sb_max_stage1
    # warm-up (the CPU has no warm-up effects; one step sizes the sample)
    t1, _, _ = sess.step(1)
    # inner iterations per step so the K timed steps take ~target seconds
    per_step = int(max(1, min(total_inner, args.ref_budget / max(args.steps, 1) / max(t1, 1e-9))))
    times, outer, ks = [], 0.0, []
    for _ in range(args.steps):
        ti, to, k = sess.step(per_step)
        times.append(ti)
        outer += to
        ks.extend(int(v) for v in k)
    sess.close()
    O.set_threads(1)
    tot = sum(times)
    val = args.steps * per_step / tot
    sample = (f"{args.steps} steps x {per_step} inner iteration(s) continuing the {cfg.name} soc schedule "
              f"(after 1 warm-up inner iteration); oracle port (the reference needs Eigen3, absent) with its "
              f"column loop on min(d, {threads}) threads and elementwise loops on {threads} threads; inner-loop "
              f"time only (set-up {sess.setup_s:.1f} s, projections {outer:.2f} s not timed)")
    return {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": DATA, "config": workload(cfg, topology_of(cfg)),
            "inner_per_step": per_step, "pcg_iters_per_inner": float(np.mean(ks)),
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                             "setup_s": sess.setup_s},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------ GPU arms ---
def per_kernel_table(kt, b, peak):
    tot_ms = sum(v[0] for v in kt.values()) or 1.0
    out = {}
    for k in ("pcg_spmv", "pcg_update", "pcg_init", "sb_pass"):
        ms, cnt = kt[k]
        if cnt:
            gbs = b[k] / (ms / cnt * 1e-3) / 1e9
            out[k] = {"avg_us": 1e3 * ms / cnt, "launches": cnt, "alg_bytes": b[k], "GB/s": gbs,
                      "frac": gbs / peak, "share": ms / tot_ms}
    return out


def run_gpu(args, rank, world, local):
    import ctypes as C

    import torch

    from paper_1612_06496_b200 import _native as N
    from paper_1612_06496_b200 import api

    dev = local if world > 1 else args.device
    cfg = load_config(args.config, seed=rank)  # replicas: one image per rank
    g, prm = cfg.graph, cfg.params
    topo = topology_of(cfg)
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    inner_per_step = prm.soc_max * prm.sb_max_stage1
    persistent = topo != "csr" and not args.no_persistent

    # ---- device-resident timing (value)
    solver = api.PfeSolver(g, prm, device=dev, use_graphs=not args.host_driven, warn=False,
                           persistent=not args.no_persistent)
    st = solver.make_state(y0)
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
    t_max = allreduce(sum(ev), world)
    rep = solver.report()
    its, _, _ = solver.pcg_log()
    k_per_inner = its[-inner_per_step:].max(axis=1)
    if persistent:
        launches_per_step = 4 * prm.soc_max + 1  # persistent kernel + 3 projection kernels per outer, rhs_quad
    else:
        launches_per_step = int((2 * k_per_inner + 4).sum() + 3 * prm.soc_max + 1)
    total_inner = allreduce(args.steps * inner_per_step, world, "sum")
    value = total_inner / t_max
    st.close()
    solver.close()

    # ---- roofline of the dominant kernel: one instrumented step after the
    # timed region, CUDA events around every launch on the solver stream
    peak, peak_src = measured_peak()
    b = algorithmic_bytes(topo, g.n, g.m, prm.dim)

    def instrumented(mode):
        s = api.PfeSolver(g, prm, device=dev, use_graphs=False, warn=False, profile=True, persistent=mode)
        ps = s.make_state(y0)
        s.run_soc(ps, prm.soc_max, prm.sb_max_stage1)  # warm (attributes, occupancy)
        s.kernel_times(reset=True)
        flush.add_(1.0)
        torch.cuda.synchronize()
        ps.reset()
        before = s.report()["inner_iterations"]
        s.run_soc(ps, prm.soc_max, prm.sb_max_stage1)
        kt = s.kernel_times()
        its_, _, _ = s.pcg_log()
        k_inner = its_[before:].max(axis=1)
        kind = s.report()["persistent_kind"]
        ps.close()
        s.close()
        return kt, k_inner, kind

    kt_m, _, _ = instrumented(False)  # one kernel per phase: the per-kernel split
    per_kernel = per_kernel_table(kt_m, b, peak)
    if persistent:
        kt_p, k_inner, kind = instrumented(True)
        ms, cnt = kt_p["sb_persistent"]
        total_b = inner_bytes(b, k_inner)
        gbs = total_b / (ms * 1e-3) / 1e9
        kname = {1: "k_sb_persistent", 2: "k_sb_resident"}.get(kind, "k_sb_persistent")
        roofline = {"bound": "hbm", "kernel": kname, "achieved": gbs, "peak": peak, "unit": "GB/s",
                    "frac": gbs / peak, "traffic": ncu_traffic(cfg.name, kname), "peak_source": peak_src,
                    "alg_bytes_per_launch": total_b / cnt, "avg_launch_us": 1e3 * ms / cnt, "launches": cnt,
                    "k_per_inner": [int(k) for k in k_inner[:prm.sb_max_stage1]],
                    "model": ("SURVEY.md §8(d): per launch (one split_bregman call = sb_max inner iterations) "
                              "sum_j B_sb + B_init + k_j B_it with B_it = 80nd + 8n + O_A, B_init = 32nd + O_A, "
                              "B_sb = 16md + 24nd + 8m, grid O_A = 8(m + n)"
                              + ("; k_sb_resident keeps the PCG state in shared memory, so its DRAM traffic is far "
                                 "below this: it is bound by grid-barrier latency" if kind == 2 else "")),
                    "timing": "CUDA events around every launch of one instrumented step after the timed region",
                    "kernels_multi_kernel_path": per_kernel}
    else:
        dom = max(per_kernel, key=lambda k: per_kernel[k]["share"])
        dk = per_kernel[dom]
        kname = {"pcg_spmv": "k_pcg_spmv", "pcg_update": "k_pcg_update", "pcg_init": "k_pcg_init",
                 "sb_pass": "k_sb_pass"}[dom]
        roofline = {"bound": "hbm", "kernel": kname, "achieved": dk["GB/s"], "peak": peak, "unit": "GB/s",
                    "frac": dk["frac"], "traffic": ncu_traffic(cfg.name, kname), "peak_source": peak_src,
                    "alg_bytes_per_launch": dk["alg_bytes"], "avg_launch_us": dk["avg_us"],
                    "model": "SURVEY.md §8(d) per-kernel contract bytes (O_A = 24m + 12n + 4 for CSR graphs)",
                    "timing": "CUDA events around every launch of one instrumented step after the timed region",
                    "kernels": per_kernel}

    # ---- end to end through the one-call C ABI with host buffers (pinned)
    gc_host = {k: pin(getattr(g, k)) for k in ("ei", "ej", "w", "degree")}
    gc = N.pfe_graph(g.n, g.m, N.iptr(gc_host["ei"]), N.iptr(gc_host["ej"]), N.dptr(gc_host["w"]),
                     N.dptr(gc_host["degree"]), *(g.grid if g.grid else (0, 0, 0)))
    pc = prm.to_c()
    xc = N.pfe_exec(dev, 1, 0, 0, 0 if args.no_persistent else 1)
    y0c = pin(np.asfortranarray(y0).reshape(-1, order="F"))
    yout = pin(np.empty(g.n * prm.dim))
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
    e2e_max = allreduce(sum(e2e_t), world)
    h2d = g.m * (4 + 4 + 8) + g.n * 8 + g.n * prm.dim * 8
    d2h = g.n * prm.dim * 8

    if rank != 0:
        return None
    cpu = cpu_baseline(cfg, args.cpu_budget) if (world == 1 and not args.no_cpu_baseline) else None
    conf = workload(cfg, topo)
    conf.update({"parallelism": f"{world} independent replicas (one image per rank)" if world > 1 else "single GPU",
                 "pcg_iters_per_inner_mean": float(k_per_inner.mean()),
                 "mode": ("persistent cooperative kernel per split_bregman call" if persistent else
                          ("host-driven" if args.host_driven else "cuda-graph (device WHILE loop)"))})
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA, "config": conf,
        "roofline": roofline, "cpu_baseline": cpu,
        "e2e": {"value": total_inner / e2e_max, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "call": "pfe_solve (solver create incl. graph upload + state + soc + Y download), pinned host buffers"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }


_PINNED = []  # owners of the pinned host buffers handed out by pin()


def pin(a):
    """A page-locked copy of a host array (torch pinned memory)."""
    import torch

    a = np.ascontiguousarray(a)
    t = torch.empty(max(1, a.size * a.itemsize), dtype=torch.uint8, pin_memory=True)
    _PINNED.append(t)
    out = t.numpy()[:a.size * a.itemsize].view(a.dtype).reshape(a.shape)
    out[...] = a
    return out


def run_bands(args, rank, world, local):
    """Strong scaling of ONE instance split across the N GPUs: row bands for
    pixel grids, vertex ranges with ghost rows for C5 (NCCL halo / ghost
    exchange + rank-ordered gathered PCG totals)."""
    import torch

    from paper_1612_06496_b200 import api

    cfg = load_config(args.config, seed=0)  # the same instance on every rank
    g, prm = cfg.graph, cfg.params
    topo = topology_of(cfg)
    y0 = api.random_embedding(g.n, prm.dim, cfg.y0_seed, g.degree)
    inner_per_step = prm.soc_max * prm.sb_max_stage1
    import torch.distributed as dist

    obj = [api.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    torch.cuda.set_device(local)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=f"cuda:{local}")
    solver = api.BandSolver(g, prm, obj[0], world, rank, device=local, warn=False)
    st = solver.make_state(y0)
    for _ in range(args.warmup):
        st.reset()
        solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)
    torch.cuda.synchronize()
    barrier(world)
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.add_(1.0)
            st.reset()
            torch.cuda.synchronize()
            barrier(world)
            solver.run_soc(st, prm.soc_max, prm.sb_max_stage1)
            times.append(solver.last_ms() * 1e-3)  # CUDA events on this rank's solver stream
    t_max = allreduce(sum(times), world)
    rep = solver.report()
    its, _, _ = solver.pcg_log()
    k_per_inner = its[-inner_per_step:].max(axis=1)
    launches_per_step = int((2 * k_per_inner + 4).sum() + 3 * prm.soc_max + 1)
    peak, peak_src = measured_peak()
    # end to end: state from host y0, solve, gathered Y back on the host
    e2e = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        s2 = solver.make_state(y0)
        solver.run_soc(s2, prm.soc_max, prm.sb_max_stage1)
        _ = s2.y
        e2e.append(time.perf_counter() - t0)
        s2.close()
    e2e_max = allreduce(sum(e2e), world)
    if rank != 0:
        return None
    conf = workload(cfg, topo)
    conf.update({"parallelism": (f"{world} row bands (NCCL halo exchange + gathered PCG totals)" if g.grid else
                                 f"{world} vertex ranges (NCCL ghost-row exchange + gathered PCG totals)"),
                 "pcg_iters_per_inner_mean": float(k_per_inner.mean()), "mode": "multi-kernel, host-driven PCG"})
    b = algorithmic_bytes(topo, g.n, g.m, prm.dim)
    tot_b = inner_bytes(b, k_per_inner)
    gbs = tot_b * args.steps / t_max / 1e9 / world
    return {
        "metric": METRIC, "value": args.steps * inner_per_step / t_max, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
        "config": conf,
        "roofline": {"bound": "hbm", "kernel": "whole inner loop (all phases)", "achieved": gbs, "peak": peak,
                     "unit": "GB/s", "frac": gbs / peak, "traffic": None, "peak_source": peak_src,
                     "model": "per GPU: (1/N) x sum_j (B_sb + B_init + k_j B_it) (SURVEY.md §8(d)) / step time",
                     "timing": "CUDA events on each rank's solver stream, max over ranks"},
        "cpu_baseline": None,
        "e2e": {"value": args.steps * inner_per_step / e2e_max, "unit": UNIT,
                "h2d_bytes_per_step": g.n * prm.dim * 8, "d2h_bytes_per_step": g.n * prm.dim * 8,
                "call": "BandSolver.make_state(y0) + run_soc + gathered state.y (graph uploaded once at solver creation)"},
        "gpu_launches": launches_per_step * args.steps,
        "clocks": clk.summary(),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--host-driven", action="store_true")
    ap.add_argument("--no-persistent", action="store_true", help="one kernel per phase instead of the "
                    "persistent cooperative kernel (grid graphs)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of 1-core inner-loop time "
                    "(at least one inner iteration) for cpu_baseline")
    ap.add_argument("--ref-budget", type=float, default=150.0, help="seconds of timed inner-loop work "
                    "for --impl reference (at least one inner iteration per step)")
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--bands", action="store_true", help="N=1: run the sharded (row-band / vertex-range) arm "
                    "with a one-rank NCCL communicator (the code path torchrun takes for N>1)")
    ap.add_argument("--replicas", action="store_true", help="N>1: independent replicas even for the "
                    "sharded configurations")
    args = ap.parse_args()
    args.config = args.config.lower()
    rank, world, local = dist_init()
    if args.impl == "reference":
        line = run_reference(args, rank, world)
    elif (world > 1 or args.bands) and args.config in SHARDED and not args.replicas:
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
