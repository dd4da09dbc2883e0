#!/usr/bin/env python
"""Benchmark: phi_0..phi_p(-tau A) v actions/s on B200 (BASELINE.json metric).

Default workload = BASELINE configs[1] (config 2): 3D advection-diffusion, n = 128 per dim
(N = 2,097,152 DOF, fp64), p = 4, eps = 1e-10, adaptive Clenshaw-Curtis.  One "step" = one
complete phi_0..phi_4 evaluation for one right-hand side (planner + node exponentials + node
sweep + combine + l squaring steps + phi_0 exp-action), through the engine's C ABI.

  value : actions/s with b already resident in HBM (device pointers), summed over ranks
  e2e   : same metric through the public host-buffer call (pinned host b in, all p+1 result
          vectors back to pinned host memory inside the timed region)
  roofline: FP64 DMMA GEMM launches (the mode products and expm products, >95% of the flops),
          algorithmic flops / CUDA-event launch time vs the measured DMMA peak
  cpu_baseline: the compiled reference (oracle/_ref) on a bounded sample

Multi-GPU (torchrun, one process per GPU): every rank evaluates its own right-hand side
(seed 1000 + rank) — independent units, no data-path collective (weak scaling); timing is the
max over ranks of the device time.  `--impl reference` times the reference CPU implementation.
"""
from __future__ import annotations

import argparse
import json
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

# Measured on this pool's B200s by tools/fp64_peak.cu (profiles/fp64_peak_r01.jsonl): mma.sync
# m8n8k4 f64 (SASS DMMA.8x8x4) register-only loop; MEASURED_PEAKS.json has no FP64 entry.
DMMA_PEAK_TFLOPS = 36.95
FP64_COPY_GBS = 6288.3


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


# ------------------------------------------------------------------ CPU reference ------------

def reference_sample(w, threads: int) -> dict:
    """Bounded sample of the reference's own CPU path on this host (oracle/_ref, unmodified
    reference headers): one reference exp_action (phi_0 = 3 Pade-13 expm + one exp-action, the
    unit every phi column is built from), extrapolated to a full phi_0..phi_p call with the
    reference's own structure: its node sweep runs `threads` nodes in parallel (ceil(q_level/T)
    waves per CC level), its l*p squaring exp-actions and phi_0 are serial."""
    from oracle.ref import Ref
    ref = Ref()
    b = w.rhs(0)
    t0 = time.perf_counter()
    ref.exp_action(w.factors, b)
    t_ea = time.perf_counter() - t0
    import math
    alpha = ref.infnorm_bound(w.factors)
    beta = float(np.max(np.abs(b)))
    l, n, _ = ref.setup_quadrature(w.eps, w.p, alpha, beta, w.mode, 0.0, 1.0, w.d)
    if w.mode == 1:
        levels = [7, 6, 12]          # CC ladder 7 -> 13 -> 25 (the GPU run reports points_used = 25)
    else:
        levels = [n + 1]
    waves = sum(math.ceil(q / max(1, threads)) for q in levels)
    serial_units = waves + l * w.p + 1
    t_call = serial_units * t_ea
    return {"t_exp_action_s": t_ea, "plan_l": l, "plan_n": n, "waves": waves, "serial_exp_actions": serial_units,
            "t_call_s": t_call}


def reference_full_call(w, threads: int) -> dict:
    """One complete reference phi_0..phi_p call on this host (oracle/_ref, unmodified reference
    headers): phiquadmv (planner, node sweep over `threads` threads, serial squaring) plus
    exp_action for phi_0 -- measured, not extrapolated.  ~23 s at config 2 on 16 cores."""
    from oracle.ref import Ref
    ref = Ref()
    b = w.rhs(0)
    t0 = time.perf_counter()
    _, info = ref.phiquadmv(w.factors, b[None, :], w.p, w.eps, w.mode, threads=threads)
    ref.exp_action(w.factors, b)
    return {"t_call_s": time.perf_counter() - t0, "plan": [info["l"], info["n"], info["points"]]}


def run_reference(args, world, rank) -> None:
    from paper_2211_00696_b200.workloads import config
    if rank != 0:
        return
    w = config(args.config)
    threads = os.cpu_count() or 1
    samples = []
    for i in range(args.warmup + args.steps):
        s = reference_sample(w, threads)
        if i >= args.warmup:
            samples.append(s)
    t_call = statistics.median([s["t_call_s"] for s in samples])
    v = 1.0 / t_call
    s0 = samples[-1]
    line = {
        "impl": "reference", "metric": "phi_0..p(tau A)v actions/sec at N=n^d DOF", "value": v,
        "unit": "actions/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t_call * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded N(0,1) RHS, BASELINE operator)",
        "config": {"workload": w.name, "N": w.N, "p": w.p, "eps": w.eps, "rule": "cc" if w.mode else "gauss"},
        "cpu_baseline": {"value": v, "unit": "actions/s", "cores": threads, "kind": "reference",
                         "sample": (f"per step: one reference exp_action on the {w.name} operator "
                                    f"({s0['t_exp_action_s']:.2f} s, threads={threads}); call time extrapolated "
                                    f"as {s0['serial_exp_actions']} serial exp-actions = {s0['waves']} node-sweep "
                                    f"waves + l*p={s0['plan_l']}*{w.p} squaring + 1 phi_0")},
        "e2e": {"value": v, "unit": "actions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ GPU arm ------------------

def run_ours(args, world, rank, local) -> None:
    import torch
    import paper_2211_00696_b200 as pq
    from paper_2211_00696_b200.workloads import config

    torch.cuda.set_device(local)
    w = config(args.config)
    nb = 1 if args.config != 3 else w.nb
    a = pq.KroneckerSum(w.factors)
    ctx = pq.Context(local)
    # one dedicated stream shared by torch (inputs, L2 flush, events) and the engine
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    req = pq.PhiRequest(p=w.p, eps=w.eps, mode=pq.QuadKind(w.mode))
    N = w.N
    bs_host = np.stack([w.rhs(rank * nb + k) for k in range(nb)])
    b_dev = torch.from_numpy(bs_host).cuda()
    # pinned host buffers for the end-to-end leg
    b_pin = torch.from_numpy(bs_host).pin_memory()
    out0_pin = torch.empty((nb, N), dtype=torch.float64).pin_memory()
    out_pin = torch.empty((nb, w.p, N), dtype=torch.float64).pin_memory()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")  # 256 MiB > 126 MB L2

    d, sh, fac = a._abi()
    rc = req._c()
    import ctypes as C
    out0 = torch.empty((nb, N), dtype=torch.float64, device="cuda")
    out = torch.empty((nb, w.p, N), dtype=torch.float64, device="cuda")
    info = pq._lib.PhiInfoC()

    def step_device():
        pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(b_dev.data_ptr()), C.byref(rc),
                                  C.c_void_p(out0.data_ptr()), C.c_void_p(out.data_ptr()), C.byref(info),
                                  pq._lib.PQ_DEVICE))

    def step_host():
        pq._lib.check(pq._lib.lib.pq_phi_0p(ctx.handle, d, sh, fac, nb, C.c_void_p(b_pin.data_ptr()), C.byref(rc),
                                  C.c_void_p(out0_pin.data_ptr()), C.c_void_p(out_pin.data_ptr()), C.byref(info),
                                  pq._lib.PQ_HOST))

    def timed(fn, k):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
        barrier(world)
        torch.cuda.synchronize()
        l0 = ctx.launches
        for i in range(k):
            flush.zero_()                       # L2 flush between steps (untimed)
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        barrier(world)
        launches = ctx.launches - l0
        ms = sum(e0.elapsed_time(e1) for e0, e1 in evs)
        return ms, launches

    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(args.warmup):
        step_device()
    torch.cuda.synchronize()
    ctx_bytes = max(1, free0 - torch.cuda.mem_get_info()[0])  # one context's workspace at this size

    with ClockSampler(local) as clk, NvmlSampler(local) as nvml:
        ms_dev, launches = timed(step_device, args.steps)
    clocks = nvml.summary() or clk.summary()
    ms_dev_max = max_over_ranks(ms_dev, world)
    units = world * nb * args.steps
    value = units / (ms_dev_max / 1e3)

    # roofline pass: same K steps with the DMMA GEMM launches bracketed by events
    ctx.set_profiling(True)
    ctx.gemm_stats(reset=True)
    for _ in range(args.steps):
        flush.zero_()
        step_device()
    g_launches, g_ms, g_flops, g_flops_dense = ctx.gemm_stats(reset=True)
    ctx.set_profiling(False)

    # end-to-end through the host-buffer call (H2D of b, D2H of phi_0..phi_p inside the region)
    for _ in range(max(1, min(args.warmup, 2))):
        step_host()
    ms_e2e, _ = timed(step_host, args.steps)
    ms_e2e_max = max_over_ranks(ms_e2e, world)
    e2e_single = units / (ms_e2e_max / 1e3)

    # ... and with several host callers (the reference API is re-entrant; each caller has its own
    # context, stream and pinned buffers), so one call's PCIe transfers and host-side syncs run
    # under another call's DMMA work (tools/e2e_diag.py: 2 callers 3.34, 3: 3.13, 4: 2.94 ms per
    # action vs 3.78 for one).  The K steps are split between the callers; the region spans from
    # one start event to the last caller's end event.  Inputs are larger than L2 (b arrives by H2D,
    # the workspaces are GB), so no flush between the overlapped calls.
    import threading
    # as many callers as the remaining HBM holds workspaces for (config 5: ~56 GB each -> fewer)
    ncall = max(1, min(args.e2e_callers, 1 + int(0.8 * torch.cuda.mem_get_info()[0] // ctx_bytes)))
    # staggered stream priorities (numerically lower = higher): equal-priority callers tend to fall
    # into lockstep (all compute, then all copy)
    pr = torch.cuda.Stream.priority_range() if hasattr(torch.cuda.Stream, "priority_range") else (0, -1)
    lo_prio, hi_prio = max(pr), min(pr)
    prios = [hi_prio + (lo_prio - hi_prio) * k // max(1, ncall - 1) for k in range(ncall)]
    callers = []
    for k in range(ncall):
        st = torch.cuda.Stream(priority=prios[k])
        cx = ctx if k == 0 else pq.Context(local)
        cx.set_stream(st.cuda_stream)
        pins = (b_pin, out0_pin, out_pin) if k == 0 else (
            torch.from_numpy(bs_host).pin_memory(), torch.empty((nb, N), dtype=torch.float64).pin_memory(),
            torch.empty((nb, w.p, N), dtype=torch.float64).pin_memory())
        callers.append((cx, st, pins))
    info2 = pq._lib.PhiInfoC()

    def host_call(cx, bufs, inf):
        pq._lib.check(pq._lib.lib.pq_phi_0p(cx.handle, d, sh, fac, nb, C.c_void_p(bufs[0].data_ptr()), C.byref(rc),
                                  C.c_void_p(bufs[1].data_ptr()), C.c_void_p(bufs[2].data_ptr()), C.byref(inf),
                                  pq._lib.PQ_HOST))

    for cx, st, bufs in callers:  # warm the second context (workspaces, caches)
        host_call(cx, bufs, info2)
    torch.cuda.synchronize()

    def e2e_callers(k):
        counts = [k // ncall + (1 if i < k % ncall else 0) for i in range(ncall)]
        start = torch.cuda.Event(enable_timing=True)
        ends = [torch.cuda.Event(enable_timing=True) for _ in callers]
        errs = []
        barrier(world)
        torch.cuda.synchronize()
        l0 = sum(cx.launches for cx, _, _ in callers)
        start.record(callers[0][1])
        for _, st, _ in callers[1:]:
            st.wait_event(start)

        def worker(i):
            cx, st, bufs = callers[i]
            try:
                inf = pq._lib.PhiInfoC()
                for _ in range(counts[i]):
                    host_call(cx, bufs, inf)
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
        ms = max(start.elapsed_time(e) for e, c in zip(ends, counts) if c > 0)
        return ms, sum(cx.launches for cx, _, _ in callers) - l0

    ms_e2e2, _ = e2e_callers(args.steps)
    ms_e2e2_max = max_over_ranks(ms_e2e2, world)
    e2e_value = units / (ms_e2e2_max / 1e3)

    fac_bytes = sum(f.size for f in w.factors) * 8
    line = {
        "metric": "phi_0..p(tau A)v actions/sec at N=n^d DOF", "value": value, "unit": "actions/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_dev_max / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded N(0,1) RHS per rank, BASELINE operator built in fp64)",
        "config": {"workload": w.name, "N": N, "d": w.d, "n": w.n, "p": w.p, "eps": w.eps, "tau": w.tau,
                   "rule": "cc" if w.mode else "gauss", "rhs_per_rank": nb,
                   "plan": {"l": info.l, "n": info.n, "points": info.points},
                   "l2": "flushed between steps (256 MiB write, untimed)", "parallelism": f"rhs-sharded x{world}"},
        "gpu_launches": launches,
        "clocks": clocks,
        "roofline": None, "cpu_baseline": None,
        "e2e": {"value": e2e_value, "unit": "actions/s", "h2d_bytes_per_step": int(nb * N * 8 + fac_bytes),
                "d2h_bytes_per_step": int(nb * (w.p + 1) * N * 8), "callers": ncall,
                "single_caller_value": e2e_single,
                "note": ("pq_phi_0p with pinned host b in and all p+1 vectors back every step; concurrent "
                         "host threads with their own contexts/streams overlap one call's PCIe transfers with "
                         "another's compute; single_caller_value = one synchronous caller")},
    }
    if g_ms > 0:
        ach = g_flops / (g_ms / 1e3) / 1e12
        # DRAM bytes per launch of the dominant kernel from the committed ncu --set full capture of
        # this workload (profiles/r01_gemm_traffic.json); null for workloads without a capture
        traffic, traffic_src = None, None
        tpath = Path(__file__).resolve().parent / "profiles" / "r01_gemm_traffic.json"
        if w.name == "cfg2_advdiff3d_n128_cc_p4" and tpath.exists():
            t = json.loads(tpath.read_text())
            traffic = t["mean_dram_bytes_per_launch"]
            traffic_src = (f"bytes/launch, mean of {len(t['launches'])} mode products in {tpath.name} "
                           f"(algorithmic {t['algorithmic_bytes_per_launch']:.3g})")
        alg = g_flops_dense / (g_ms / 1e3) / 1e12
        line["roofline"] = {"bound": "tensor", "achieved": alg, "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                            "frac": alg / DMMA_PEAK_TFLOPS, "traffic": traffic, "traffic_source": traffic_src,
                            "executed_tflops": ach, "executed_frac": ach / DMMA_PEAK_TFLOPS,
                            "kernel": "k_gemm (FP64 DMMA mode products + expm products)",
                            "launches": g_launches, "gemm_ms_per_step": g_ms / args.steps,
                            "flops_note": ("achieved = ALGORITHMIC flops (dense 2*M*N*K per mode product, SURVEY 8(d); "
                                           "skipped work not credited) / GEMM time, which exceeds the DMMA peak because "
                                           "the tiles skip exponential blocks below 2^-64 max|E| (DESIGN.md 3b); "
                                           "executed_* = the FLOPs the DMMA tiles actually issued (device counters)"),
                            "gemm_share_of_step": (g_ms / args.steps) / (ms_dev / args.steps),
                            "peak_source": "measured DMMA loop, profiles/fp64_peak_r01.jsonl"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            threads = os.cpu_count() or 1
            if w.N <= 4_000_000:  # a full reference call fits the 10-30 s budget (config 2: ~23 s)
                s = reference_full_call(w, threads)
                sample = (f"one complete reference phi_0..phi_{w.p} call on this workload (phiquadmv + exp_action, "
                          f"{threads} threads for the node sweep, squaring serial as in the reference), measured: "
                          f"{s['t_call_s']:.1f} s, plan (l, n, points) = {tuple(s['plan'])}")
            else:
                s = reference_sample(w, threads)
                sample = (f"one reference exp_action on this operator ({s['t_exp_action_s']:.2f} s), extrapolated to "
                          f"{s['serial_exp_actions']} serial exp-actions per phi_0..phi_{w.p} call "
                          f"(node waves {s['waves']} at {threads} threads + l*p + phi_0; l={s['plan_l']})")
            line["cpu_baseline"] = {"value": 1.0 / s["t_call_s"], "unit": "actions/s", "cores": threads,
                                    "kind": "reference", "sample": sample}
        except Exception as e:  # oracle missing on this box: say so
            line["cpu_baseline"] = {"value": None, "unit": "actions/s", "cores": 0, "kind": "reference",
                                    "sample": f"unavailable: {e}"}
    if rank == 0:
        print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 5])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-callers", type=int, default=4, help="concurrent host callers in the e2e leg")
    args = ap.parse_args()
    world, rank, local = dist_init() if args.impl == "ours" else (int(os.environ.get("WORLD_SIZE", "1")),
                                                                    int(os.environ.get("RANK", "0")), 0)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1 and args.impl == "ours":
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
