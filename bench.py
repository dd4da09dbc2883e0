#!/usr/bin/env python
"""Benchmark: phi_0..phi_p(-tau A) v actions/s on B200 (BASELINE.json metric).

Default workload = BASELINE configs[1] (config 2): 3D advection-diffusion, n = 128 per dim
(N = 2,097,152 DOF, fp64), p = 4, eps = 1e-10, adaptive Clenshaw-Curtis.  One "step" = one
complete phi_0..phi_4 evaluation for one right-hand side (planner + node exponentials + node
sweep + combine + l squaring steps + phi_0 exp-action), through the engine's C ABI.  Every step
gets a FRESH seeded right-hand side (seed 1000 + i for step i, warm-up steps first), so nothing
the host memoises per b survives from one step to the next.

  value : actions/s with the step's b already resident in HBM (device pointers), all ranks
  e2e   : same metric through the public host-buffer call (pinned host b in, all p+1 result
          vectors back to pinned host memory inside the timed region)
  roofline: FP64 DMMA GEMM launches (mode products + expm products): EXECUTED flops / CUDA-event
          launch time vs the measured DMMA peak; the dense-equivalent rate is reported beside it
  cpu_baseline: the compiled reference (oracle/_ref) on this host: one complete call (config 2)

`--impl reference` times the reference's own CPU path (oracle/_ref: the unmodified reference
headers) with all host threads: for configs 1 and 2 every step is one COMPLETE reference
phiquadmv + exp_action call on that step's right-hand side (no extrapolation); it never loads
libpq_b200.so.  Config 4 (`--config 4`, ETDRK4 Allen-Cahn) reports ETDRK4 time steps/s.

Multi-GPU (torchrun, one process per GPU): `--shard rhs` (default for N > 1 until the node
sharded path is selected with `--shard nodes`): every rank evaluates its own right-hand sides --
independent units, no data-path collective (weak scaling); timing is the max over ranks of the
device time.
"""
from __future__ import annotations

import argparse
import importlib.util
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# Measured on this pool's B200s by tools/fp64_peak.cu (profiles/fp64_peak_r02.jsonl, best of 3 runs
# x 9 launch shapes; r01: 36.95): mma.sync m8n8k4 f64 (SASS DMMA.8x8x4) register-only loop at
# 1965 MHz = 148 SMs x 4 SMSPs x 32 flop/clk; MEASURED_PEAKS.json has no FP64 entry.
DMMA_PEAK_TFLOPS = 37.15
FP64_COPY_GBS = 6288.3
METRIC = "phi_0..p(tau A)v actions/sec at N=n^d DOF"


def load_workloads():
    """paper_2211_00696_b200/workloads.py loaded by path: importing it through the package would
    run the package __init__, which loads libpq_b200.so (the reference arm must not)."""
    spec = importlib.util.spec_from_file_location("_pq_workloads", ROOT / "paper_2211_00696_b200" / "workloads.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod  # dataclasses resolve their module through sys.modules
    spec.loader.exec_module(mod)
    return mod


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return {}


class NvmlSampler:
    """SM clock and clock-event reasons polled through NVML every ~2 ms on a host thread, strictly
    inside the timed region (a short region holds no nvidia-smi sample at its 200 ms period)."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, device: int):
        self.device, self.rows, self.max_mhz, self.ok = device, [], None, False
        self.stop = None

    def __enter__(self):
        import threading
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            self.stop = threading.Event()

            def poll():
                while not self.stop.is_set():
                    try:
                        self.rows.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                          nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
                    except Exception:
                        pass
                    self.stop.wait(0.002)

            self.thread = threading.Thread(target=poll, daemon=True)
            self.thread.start()
            self.ok = True
        except Exception:
            self.ok = False
        return self

    def __exit__(self, *exc):
        if self.ok:
            self.stop.set()
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        if not self.ok or not self.rows:
            return None
        import pynvml as nv
        reasons = sorted({name for _, bits in self.rows for name, const in self.REASONS
                          if hasattr(nv, const) and bits & getattr(nv, const)})
        return {"sm_mhz": statistics.median(r[0] for r in self.rows), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(self.rows), "source": "NVML, 2 ms, timed region"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.f = None

    def __enter__(self):
        try:
            self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        rows = []
        try:
            for line in Path(self.f.name).read_text().splitlines():
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if _backend() == "gloo":
            # plumbing check only (tests/test_gpu_bench_contract.py): ranks share the visible GPUs; the
            # RHS-sharded data path has no collective, gloo carries the barrier and the max-over-ranks
            local = local % torch.cuda.device_count()
            torch.cuda.set_device(local)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def _backend() -> str:
    return os.environ.get("PQ_BENCH_BACKEND", "nccl")


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cpu" if _backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()




# ------------------------------------------------------------------ shared config -----------

def bench_config(w, args, world: int) -> dict:
    """The `config` object BOTH arms print (identical dict for the same flags)."""
    cfg = {"workload": w.name, "N": w.N, "d": w.d, "n": w.n, "p": w.p, "eps": w.eps, "tau": w.tau,
           "rule": "cc" if w.mode else "gauss", "rhs_per_step": w.nb if args.config == 3 else 1,
           "rhs": "fresh seeded N(0,1) b per step: seed 1000 + i (warm-up steps first), numpy PCG64",
           "l2": "flushed between steps (256 MiB write, untimed)",
           "parallelism": f"{args.shard}-sharded x{world}"}
    if args.config == 4:
        cfg.update({"rhs_per_step": 1, "rhs": "u0 ~ U[-0.9, 0.9] seed 2024; one step = one ETDRK4 time step (dt = tau)",
                    "steps_per_integration": args.etd_steps})
    return cfg


def step_seeds(args, rank: int, nb: int) -> list:
    """RHS seed indices per bench step (warm-up first), for this rank."""
    per = args.warmup + args.steps
    return [[(rank * per + i) * nb + k for k in range(nb)] for i in range(per)]


# ------------------------------------------------------------------ CPU reference ------------

def reference_phi_call(ref, w, b, threads: int) -> dict:
    """One complete reference phi_0..phi_p call (oracle/_ref, unmodified reference headers):
    phiquadmv (planner, node sweep over `threads` threads, serial squaring, phiaction.hpp:307-346)
    plus exp_action for phi_0 (kron.hpp:123-128) -- measured, not extrapolated."""
    t0 = time.perf_counter()
    _, info = ref.phiquadmv(w.factors, b[None, :], w.p, w.eps, w.mode, threads=threads)
    ref.exp_action(w.factors, b)
    return {"t_call_s": time.perf_counter() - t0, "plan": [info["l"], info["n"], info["points"]]}


def reference_extrapolated(ref, w, b, threads: int) -> dict:
    """Configs 3 and 5 only (a complete reference call takes 10 min .. hours): one reference
    exp_action on the operator, scaled by the reference's own structure -- node-sweep waves over
    `threads` threads + l*p serial squaring exp-actions + phi_0.  Labelled as an extrapolation."""
    t0 = time.perf_counter()
    ref.exp_action(w.factors, b)
    t_ea = time.perf_counter() - t0
    alpha = ref.infnorm_bound(w.factors)
    beta = float(np.max(np.abs(b)))
    l, n, _ = ref.setup_quadrature(w.eps, w.p, alpha, beta, w.mode, 0.0, 1.0, w.d)
    waves = math.ceil((n + 1) / max(1, threads))
    units = waves + l * w.p + 1
    return {"t_call_s": units * t_ea, "t_exp_action_s": t_ea, "plan": [l, n, n + 1], "units": units}


def run_reference(args, world, rank) -> None:
    if rank != 0:
        return
    from oracle.ref import Ref
    W = load_workloads()
    w = W.config(args.config)
    ref = Ref()
    threads = os.cpu_count() or 1
    cfg = bench_config(w, args, world)
    if args.config == 4:
        # bounded sample: one reference integrate over `ref_etd_steps` ETDRK4 steps per bench step
        u0 = W.allen_cahn_u0(w.N)
        m = args.ref_etd_steps
        times = []
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            ref.integrate(w.A, 1, u0, 0.0, m * w.tau, m, 3, eps=w.eps, threads=threads)
            if i >= args.warmup:
                times.append(time.perf_counter() - t0)
        v = args.steps * m / sum(times)
        sample = (f"per bench step: reference integrate (integrators.hpp:193) of {m} ETDRK4 steps (Allen-Cahn, "
                  f"n={w.n}, tableau as ExpRKTableau, {threads} threads), measured; value = time steps/s")
        unit = "ETDRK4 steps/s"
        ms = sum(times) / len(times) * 1e3
    else:
        seeds = step_seeds(args, 0, 1)
        times, plans = [], set()
        full = args.config in (1, 2)
        for i, s in enumerate(seeds):
            b = w.rhs(s[0])
            r = reference_phi_call(ref, w, b, threads) if full else reference_extrapolated(ref, w, b, threads)
            if i >= args.warmup:
                times.append(r["t_call_s"])
                plans.add(tuple(r["plan"]))
        nb = w.nb if args.config == 3 else 1
        v = args.steps * nb / sum(times) if full else nb / statistics.median(times)
        unit = "actions/s"
        ms = sum(times) / len(times) * 1e3
        sample = (f"every bench step one COMPLETE reference phiquadmv + exp_action call on that step's fresh b "
                  f"({threads} threads for the node sweep; squaring serial as in the reference), measured; "
                  f"plans (l, n, points) seen: {sorted(plans)}" if full else
                  f"extrapolated: one reference exp_action per step scaled to {r['units']} serial exp-actions "
                  f"(node waves at {threads} threads + l*p + phi_0) per RHS, x{nb} RHS")
    line = {
        "impl": "reference", "metric": METRIC if args.config != 4 else "ETDRK4 time steps/s (config 4)",
        "value": v, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak" if args.shard == "rhs" else "strong",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded inputs, BASELINE operator built in fp64)", "config": cfg,
        "cpu_baseline": {"value": v, "unit": unit, "cores": threads, "kind": "reference", "sample": sample},
        "e2e": {"value": v, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm ------------------

def roofline_line(ctx, steps: int, ms_step_dev: float, w, kstats=None) -> dict:
    """DMMA roofline of the GEMM launches recorded while profiling (ctx.gemm_stats), plus the HBM
    roofline of the streaming kernels (ctx.kernel_stats) when available."""
    g_launches, g_ms, g_flops, g_flops_dense = ctx.gemm_stats(reset=True)
    if g_ms <= 0:
        return None
    ach = g_flops / (g_ms / 1e3) / 1e12
    dense = g_flops_dense / (g_ms / 1e3) / 1e12
    traffic, traffic_src = None, None
    tpath = ROOT / "profiles" / "r02_gemm_traffic.json"
    if not tpath.exists():
        tpath = ROOT / "profiles" / "r01_gemm_traffic.json"
    if w.name == "cfg2_advdiff3d_n128_cc_p4" and tpath.exists():
        t = json.loads(tpath.read_text())
        traffic = t["mean_dram_bytes_per_launch"]
        traffic_src = (f"DRAM bytes/launch, mean of {len(t['launches'])} node-sweep mode products in {tpath.name} "
                       f"(ncu --set full; algorithmic {t['algorithmic_bytes_per_launch']:.3g})")
    ro = {"bound": "tensor", "achieved": ach, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
          "frac": ach / DMMA_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
          "kernel": ("k_gemm band tiles + k_slab12 (FP64 DMMA mode products) + expm products, all launches "
                     "of the step"),
          "achieved_note": ("EXECUTED flops: each warp adds 2*rows*cols*4 per DMMA k4 step it issued to a device "
                            "counter; exponential blocks and 8-row groups below 2^-64 of their max are skipped "
                            "(DESIGN.md 3b) and not counted -- since the fine gating the tiles are bound by operand "
                            "streaming, so this fraction is below the dense-equivalent one"),
          "dense_equiv_tflops": dense, "dense_equiv_frac": dense / DMMA_PEAK_TFLOPS,
          "dense_equiv_note": "2*M*N*K of the same launches (the reference's dense mode products) / the same time",
          "launches_per_step": g_launches / steps, "gemm_ms_per_step": g_ms / steps,
          "gemm_share_of_step": (g_ms / steps) / ms_step_dev if ms_step_dev > 0 else None,
          "peak_source": "measured DMMA loop, profiles/fp64_peak_r02.jsonl (MEASURED_PEAKS.json has no FP64 entry)"}
    if kstats:
        hbm = load_peaks().get("hbm_gbs") or FP64_COPY_GBS
        rows = {}
        for name, s in sorted(kstats.items()):
            if s["ms"] <= 0:
                continue
            gbs = s["bytes"] / (s["ms"] / 1e3) / 1e9
            rows[name] = {"launches_per_step": s["launches"] / steps, "ms_per_step": s["ms"] / steps,
                          "GB/s": gbs, "frac": gbs / hbm}
        ro["hbm_kernels"] = {"peak_GBps": hbm, "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)",
                             "kernels": rows, "bytes_note": "algorithmic bytes: every vector read/written once"}
    return ro


def cpu_baseline_line(w, args) -> dict:
    threads = os.cpu_count() or 1
    try:
        from oracle.ref import Ref
        ref = Ref()
        if w.N <= 4_000_000 and args.config in (1, 2):
            s = reference_phi_call(ref, w, w.rhs(0), threads)
            sample = (f"one complete reference phi_0..phi_{w.p} call on this workload (phiquadmv + exp_action, "
                      f"{threads} threads for the node sweep, squaring serial as in the reference), measured: "
                      f"{s['t_call_s']:.1f} s, plan (l, n, points) = {tuple(s['plan'])}")
        else:
            s = reference_extrapolated(ref, w, w.rhs(0), threads)
            sample = (f"one reference exp_action on this operator ({s['t_exp_action_s']:.2f} s), extrapolated to "
                      f"{s['units']} serial exp-actions per phi_0..phi_{w.p} call")
        return {"value": 1.0 / s["t_call_s"], "unit": "actions/s", "cores": threads, "kind": "reference",
                "sample": sample}
    except Exception as e:  # oracle missing on this box: say so
        return {"value": None, "unit": "actions/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}


def _pool(host_rows: list, nbytes_each: int, budget: int):
    """How many distinct per-step inputs to keep: all of them when they fit `budget` bytes, else
    cycle through as many as fit (at least 2, so consecutive steps never share b)."""
    return max(2, min(len(host_rows), budget // max(1, nbytes_each)))


def run_ours_phi(args, world, rank, local) -> None:
    import ctypes as C
    import threading

    import torch
    import paper_2211_00696_b200 as pq

    W = load_workloads()
    torch.cuda.set_device(local)
    w = W.config(args.config)
    nb = w.nb if args.config == 3 else 1
    N = w.N
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(local)
    # one dedicated stream shared by torch (inputs, L2 flush, events) and the engine
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    nodes = args.shard == "nodes"
    comm = None
    if nodes:
        # one phi call spans all ranks: quadrature nodes dealt round-robin, node vectors moved
        # into x-slabs, distributed squaring (csrc/dist.cpp); every rank passes the same b
        from paper_2211_00696_b200 import sharded as S
        if world == 1:
            comm = S.Communicator.single()
        elif args.transport == "peer":
            comm = S.Communicator.peer(ctx)  # flips fused into the mode products (CUDA IPC / NVLink stores)
        elif _backend() == "gloo" or args.transport == "host":
            comm = S.Communicator.host()  # plumbing check: ranks share one GPU, collectives via the host
        else:
            comm = S.Communicator.nccl(ctx)
        sb, se = S.slab_range(a.shape(), world, rank)
    seeds = step_seeds(args, 0 if nodes else rank, nb)
    per_step = nb * N * 8
    free = torch.cuda.mem_get_info()[0]
    npool = _pool(seeds, per_step, min(8 << 30, free // 6))
    hosts = [np.stack([w.rhs(s) for s in seeds[i]]) for i in range(len(seeds))]
    b_dev = [torch.from_numpy(hosts[i]).cuda() for i in range(npool)]
    npin = _pool(seeds, per_step, 4 << 30)
    b_pin = [torch.from_numpy(hosts[i]).pin_memory() for i in range(npin)]
    NO = (se - sb) if nodes else N  # result length per column on this rank (slab or full vector)
    out0_pin = torch.empty((nb, NO), dtype=torch.float64).pin_memory()
    out_pin = torch.empty((nb, w.p, NO), dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    d, sh, fac = a._abi()
    rc = req._c()
    out0 = torch.empty((nb, NO), dtype=torch.float64, device="cuda")
    out = torch.empty((nb, w.p, NO), dtype=torch.float64, device="cuda")
    info = pq._lib.PhiInfoC()
    plans = set()

    def call(cx, b, o0, o, inf, space):
        if nodes:
            pq._lib.check(pq._lib.lib.pq_phiquadmv_dist(cx.handle, comm.handle, d, sh, fac, nb, C.c_void_p(b),
                                                        C.byref(rc), C.c_void_p(o0), C.c_void_p(o), C.byref(inf),
                                                        space, 0))
        else:
            pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, nb, C.c_void_p(b), C.byref(rc), C.c_void_p(o0),
                                                C.c_void_p(o), C.byref(inf), space))

    def step_device(i):
        call(ctx, b_dev[i % npool].data_ptr(), out0.data_ptr(), out.data_ptr(), info, pq._lib.PQ_DEVICE)
        plans.add((info.l, info.n, info.points))

    def host_call(cx, i, bufs, inf):
        call(cx, b_pin[i % npin].data_ptr(), bufs[0].data_ptr(), bufs[1].data_ptr(), inf, pq._lib.PQ_HOST)

    def timed(fn, first, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier(world)
        torch.cuda.synchronize()
        l0 = ctx.launches
        for i in range(k):
            flush.zero_()                       # L2 flush between steps (untimed)
            evs[i][0].record(stream)
            fn(first + i)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return sum(e0.elapsed_time(e1) for e0, e1 in evs), ctx.launches - l0

    free0 = torch.cuda.mem_get_info()[0]
    for i in range(args.warmup):
        step_device(i)
    torch.cuda.synchronize()
    ctx_bytes = max(1, free0 - torch.cuda.mem_get_info()[0])  # one context's workspace at this size

    with ClockSampler(local) as clk, NvmlSampler(local) as nvml:
        ms_dev, launches = timed(step_device, args.warmup, args.steps)
    clocks = nvml.summary() or clk.summary()
    ms_dev_max = max_over_ranks(ms_dev, world)
    units = (1 if nodes else world) * nb * args.steps  # node sharding: the ranks share each action
    value = units / (ms_dev_max / 1e3)

    # roofline pass: the same K steps (same b's) with every DMMA GEMM and streaming kernel bracketed
    ctx.set_profiling(True)
    ctx.gemm_stats(reset=True)
    ctx.kernel_stats(reset=True)
    for i in range(args.steps):
        flush.zero_()
        step_device(args.warmup + i)
    kst = ctx.kernel_stats(reset=True)
    roof = roofline_line(ctx, args.steps, ms_dev / args.steps, w, kst)
    ctx.set_profiling(False)

    # end-to-end through the host-buffer call (H2D of b, D2H of phi_0..phi_p inside the region)
    for i in range(max(1, min(args.warmup, 2))):
        host_call(ctx, i, (out0_pin, out_pin), info)
    torch.cuda.synchronize()
    ms_e2e, _ = timed(lambda i: host_call(ctx, i, (out0_pin, out_pin), info), args.warmup, args.steps)
    ms_e2e_max = max_over_ranks(ms_e2e, world)
    e2e_single = units / (ms_e2e_max / 1e3)

    # ... and with several host callers (the reference API is re-entrant; each caller has its own
    # context, stream and pinned result buffers), so one call's PCIe transfers and host-side syncs
    # run under another call's DMMA work.  The K steps (each its own fresh b) are split between the
    # callers; the region spans from one start event to the last caller's end event.  Inputs are
    # larger than L2 (b arrives by H2D, the workspaces are GB), so no flush between the calls.
    ncall = max(1, min(args.e2e_callers, 1 + int(0.8 * torch.cuda.mem_get_info()[0] // ctx_bytes)))
    if nodes:
        ncall = 1  # one communicator: distributed calls must not interleave their collectives
    pr = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    lo_prio, hi_prio = max(pr), min(pr)
    prios = [hi_prio + (lo_prio - hi_prio) * k // max(1, ncall - 1) for k in range(ncall)]
    callers = []
    for k in range(ncall):
        st = torch.cuda.Stream(priority=prios[k])
        cx = ctx if k == 0 else pq.Context(local)
        cx.set_stream(st.cuda_stream)
        bufs = (out0_pin, out_pin) if k == 0 else (torch.empty((nb, NO), dtype=torch.float64).pin_memory(),
                                                   torch.empty((nb, w.p, NO), dtype=torch.float64).pin_memory())
        callers.append((cx, st, bufs))
    for k, (cx, st, bufs) in enumerate(callers):  # warm the other contexts (workspaces, caches)
        host_call(cx, k, bufs, pq._lib.PhiInfoC())
    torch.cuda.synchronize()

    def e2e_callers(k):
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in callers]
        mine = [[args.warmup + j for j in range(k) if j % ncall == i] for i in range(ncall)]
        errs = []
        barrier(world)
        torch.cuda.synchronize()
        start.record(callers[0][1])
        for _, st, _ in callers[1:]:
            st.wait_event(start)

        def worker(i):
            cx, st, bufs = callers[i]
            try:
                inf = pq._lib.PhiInfoC()
                for j in mine[i]:
                    host_call(cx, j, bufs, inf)
                ends[i].record(st)
            except Exception as e:  # pragma: no cover - surfaced below
                errs.append(e)

        ths = [threading.Thread(target=worker, args=(i,)) for i in range(len(callers))]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        if errs:
            raise errs[0]
        torch.cuda.synchronize()
        barrier(world)
        return max(start.elapsed_time(e) for e, m in zip(ends, mine) if m)

    if nodes:
        comm.stats(reset=True)
    # at least 4 calls per caller: with fewer, the simultaneous start and the last caller's tail
    # dominate the region (config 2, 6 callers: 385-409 actions/s over 10 calls, 438 over 24)
    k_multi = max(args.steps, 4 * ncall)
    # the region is short (tens of ms at config 2) and runs on shared host cores: three repetitions,
    # the MEDIAN is reported and all three are listed (one noisy box measured 406 / 518 / 518)
    reps_ms = [max_over_ranks(e2e_callers(k_multi), world) for _ in range(1 if nodes else 3)]
    ms_e2e2_max = sorted(reps_ms)[len(reps_ms) // 2]
    comm_bytes = comm.stats(reset=True)[0] / args.steps if nodes else None
    e2e_multi = units * k_multi / args.steps / (ms_e2e2_max / 1e3)
    # a deployment runs as many host callers as pays: small problems (config 1, ~0.2 ms per call)
    # are host-latency bound and lose to thread contention with 4 callers; report the better of
    # the two measured configurations and say which
    e2e_value, e2e_callers = (e2e_multi, ncall) if e2e_multi >= e2e_single else (e2e_single, 1)

    line = {
        "metric": METRIC, "value": value, "unit": "actions/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev_max / args.steps,
        "higher_is_better": True, "scaling": "strong" if nodes else "weak", "vs_baseline": None, "dtype": "f64",
        "data": ("synthetic (fresh seeded N(0,1) RHS per step" + ("" if nodes else " and rank")
                 + ", BASELINE operator built in fp64)"),
        "config": bench_config(w, args, world),
        "plans": sorted(list(p) for p in plans),
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": roof, "cpu_baseline": None,
        "e2e": {"value": e2e_value, "unit": "actions/s", "h2d_bytes_per_step": int(nb * N * 8),
                "d2h_bytes_per_step": int(nb * (w.p + 1) * NO * 8), "callers": e2e_callers,
                "single_caller_value": e2e_single, "multi_caller_value": e2e_multi, "multi_callers": ncall,
                "multi_caller_calls": k_multi,
                "multi_caller_reps": [units * k_multi / args.steps / (m / 1e3) for m in reps_ms],
                "distinct_rhs": {"device": npool, "pinned_host": npin},
                "note": ("pq_phi_0p with pinned host b in and all p+1 vectors back every step; concurrent "
                         "host threads with their own contexts/streams overlap one call's PCIe transfers with "
                         "another's compute; value = the better of single_caller_value (one synchronous caller) "
                         "and multi_caller_value (multi_callers threads sharing multi_caller_calls calls, at least 4 "
                         "each; the median of the repetitions listed in multi_caller_reps), `callers` says which; the operator's "
                         "factors are uploaded once (bit-identical factors are not re-copied) and not counted")},
    }
    if nodes:
        line["distributed"] = {"transport": ("peer (fused IPC stores)" if args.transport == "peer" else
                                              "host (gloo)" if (world > 1 and _backend() == "gloo") else "nccl"),
                               "slab": [sb, se], "bytes_sent_per_step_rank0": comm_bytes,
                               "outputs": "x-slabs per rank (gather=0)"}
        comm.close()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(w, args)
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_ours_etd(args, world, rank, local) -> None:
    """Config 4: ETDRK4 on Allen-Cahn (n = 128, dt = 1e-3).  One bench step = one integrate() of
    `--etd-steps` time steps (the whole config-4 run at the default 100) from u0 resident in HBM;
    value = ETDRK4 time steps per second (all ranks: independent runs, weak)."""
    import ctypes as C

    import torch
    import paper_2211_00696_b200 as pq

    W = load_workloads()
    torch.cuda.set_device(local)
    w = W.config(4)
    N, m = w.N, args.etd_steps
    a = pq.KroneckerSum(w.A)
    ctx = pq.Context(local)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    u0h = W.allen_cahn_u0(N, seed=2024 + rank)
    u0 = torch.from_numpy(u0h).cuda()
    u0_pin = torch.from_numpy(u0h).pin_memory()
    u_out = torch.empty(N, dtype=torch.float64, device="cuda")
    u_pin = torch.empty(N, dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    tab = pq.etdrk4_tableau()
    tc, tkeep = tab._c()
    src, skeep = pq.phiquad._source(("cubic", 1.0, -1.0))
    base = pq.PhiRequest(eps=w.eps)._c()
    d, sh, fac = a._abi()
    calls = C.c_int()

    def run(space):
        ui, uo = (u0, u_out) if space == pq._lib.PQ_DEVICE else (u0_pin, u_pin)
        pq._lib.check(pq._lib.lib.pq_integrate(ctx.handle, d, sh, fac, C.byref(src), C.c_void_p(ui.data_ptr()),
                                               0.0, m * w.tau, m, C.byref(tc), C.byref(base),
                                               C.c_void_p(uo.data_ptr()), C.byref(calls), space))

    def timed(space, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier(world)
        torch.cuda.synchronize()
        l0 = ctx.launches
        for i in range(k):
            flush.zero_()
            evs[i][0].record(stream)
            run(space)
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier(world)
        return sum(e0.elapsed_time(e1) for e0, e1 in evs), ctx.launches - l0

    for _ in range(args.warmup):
        run(pq._lib.PQ_DEVICE)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk, NvmlSampler(local) as nvml:
        ms_dev, launches = timed(pq._lib.PQ_DEVICE, args.steps)
    clocks = nvml.summary() or clk.summary()
    ms_max = max_over_ranks(ms_dev, world)
    value = world * args.steps * m / (ms_max / 1e3)
    ctx.set_profiling(True)
    ctx.gemm_stats(reset=True)
    ctx.kernel_stats(reset=True)
    for _ in range(args.steps):
        flush.zero_()
        run(pq._lib.PQ_DEVICE)
    kst = ctx.kernel_stats(reset=True)
    roof = roofline_line(ctx, args.steps * m, ms_dev / (args.steps * m), w, kst)
    ctx.set_profiling(False)
    run(pq._lib.PQ_HOST)
    ms_e2e, _ = timed(pq._lib.PQ_HOST, args.steps)
    e2e = world * args.steps * m / (max_over_ranks(ms_e2e, world) / 1e3)
    line = {
        "metric": "ETDRK4 time steps/s (config 4)", "value": value, "unit": "ETDRK4 steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (u0 ~ U[-0.9,0.9] seeded, Allen-Cahn operator built in fp64)",
        "config": bench_config(w, args, world), "phi_calls_per_integration": calls.value,
        "gpu_launches": launches, "clocks": clocks, "roofline": roof, "cpu_baseline": None,
        "e2e": {"value": e2e, "unit": "ETDRK4 steps/s", "h2d_bytes_per_step": N * 8, "d2h_bytes_per_step": N * 8,
                "note": "pq_integrate with pinned host u0 in and u back every bench step"},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle.ref import Ref
            ref = Ref()
            threads = os.cpu_count() or 1
            k = args.ref_etd_steps
            t0 = time.perf_counter()
            ref.integrate(w.A, 1, u0h, 0.0, k * w.tau, k, 3, eps=w.eps, threads=threads)
            t = time.perf_counter() - t0
            line["cpu_baseline"] = {"value": k / t, "unit": "ETDRK4 steps/s", "cores": threads, "kind": "reference",
                                    "sample": f"reference integrate of {k} ETDRK4 steps, measured ({t:.1f} s)"}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": "ETDRK4 steps/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--shard", default=None, choices=["rhs", "nodes"],
                    help="N > 1: rhs = independent right-hand sides per rank (weak scaling; default for the CC "
                         "configs 2 and 4), nodes = one action across all ranks (csrc/dist.cpp, strong scaling; "
                         "default for the Gauss configs 1, 3, 5)")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "peer", "host"],
                    help="--shard nodes: NCCL packed exchanges, peer (flips fused into the mode products "
                         "through CUDA IPC), or the host transport")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-callers", type=int, default=6, help="concurrent host callers in the e2e leg")
    ap.add_argument("--etd-steps", type=int, default=100, help="config 4: ETDRK4 steps per bench step")
    ap.add_argument("--ref-etd-steps", type=int, default=2, help="config 4: reference ETDRK4 steps per sample")
    args = ap.parse_args()
    if args.shard is None:
        args.shard = "nodes" if (args.config in (1, 3, 5) and int(os.environ.get("WORLD_SIZE", "1")) > 1) else "rhs"
    if args.impl == "reference":
        world, rank = int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0"))
        run_reference(args, world, rank)
        return
    world, rank, local = dist_init()
    if args.config == 4:
        run_ours_etd(args, world, rank, local)
    else:
        run_ours_phi(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
