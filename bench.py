#!/usr/bin/env python
"""Benchmark of the vertex-patch smoother hot path (arXiv 2412.05082) -- one JSON line.

Workload (BASELINE.json configs[1] / SURVEY.md §8d cfg2): 2D unit square, Q_k C0IP with
k = --degree (default 4), N_k cells per axis so that (kN-1)^2 ~ 16.7M DoFs, FP64, one B200.
A *step* is one additive vertex-patch smoothing application: residual
r = b - A x with the matrix-free C0IP operator, per-patch gather, approximate FDM local solve
(S^T, Lambda^-1, S per axis) and scatter-add, all on device.

value  = DoFs x ranks / (max over ranks of the device time per step), GDoF/s.
e2e    = the same step through the C ABI with host buffers: x, b copied from pinned host
         memory to the device and x' back, inside the timed region.
Extras: matvec GDoF/s on the same mesh, per-kernel roofline of the dominant kernel, an MG-PCG
time-to-solve (FP64 vs FP32 V-cycle, nested mesh) and the CPU oracle baseline.

Multi-GPU (torchrun, --gpus N): weak scaling on a y-slab decomposition of a global mesh with
~16.7M DoFs per GPU; every step exchanges ghost rows between neighbours (NCCL send/recv) before
the slab smoothing step; timing is the max over ranks.
--impl reference: times the CPU oracle (oracle/) on a bounded sample of the same workload.
"""
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

from c0ip_inputs import CFG2_CELLS, CFG4_CELLS, random_xb  # noqa: E402

METRIC = "smoother & C0IP matvec GDoF/s; MG-PCG time-to-solve, FP64 vs mixed precision"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            d = json.load(fh)
        return d.get("hbm_gbs", 6650.0), d.get("sm_max_mhz", 1965.0), "measured"
    except Exception:
        return 6650.0, 1965.0, "fallback"


def _alu_peaks():
    """Measured DFMA / FFMA / DMMA throughput on this B200 pool (tools/alu_peaks.cu, committed as
    profiles/alu_peaks.json), else the unit-count derivation 148 SMs x 64 (FP64) / 128 (FP32) FMA/clk."""
    try:
        with open(os.path.join(ROOT, "profiles", "alu_peaks.json")) as fh:
            return json.load(fh)
    except Exception:
        return None


def fp64_peak_tflops(mhz):
    """FP64 peak at the given SM clock: measured DFMA rate (= measured DMMA rate) rescaled from the
    clock it was measured at; fallback 148 x 64 FMA/clk x 2 flop."""
    p = _alu_peaks()
    if p:
        return max(p["dfma_tflops"], p.get("dmma_m8n8k4_tflops", 0.0)) * mhz / p["dfma_sm_mhz"]
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


def fp32_peak_tflops(mhz):
    p = _alu_peaks()
    if p:
        return p["ffma_tflops"] * mhz / p["ffma_sm_mhz"]
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


# algorithmic work per DoF of the fused 2D kernels; FP64 bytes
def flops_residual_2d(k):
    # x-stage B^ (avg 3k+2 nonzeros), L^, M^ (avg k+2) and the same on the y-stage, 2 flop/MAC
    per = (3 * k + 2) + 2 * (k + 2)
    return 2.0 * 2 * per


def flops_residual_3d(k):
    # x-stage (B, L, M), y-stage (6 contractions), z-stage (3): MACs with banded averages 3k+2 / k+2
    return 2.0 * ((3 * k + 2) + 2 * (k + 2) + (3 * k + 2) + 5 * (k + 2) + (3 * k + 2) + 2 * (k + 2))


def flops_fdm_3d(k):
    np_ = 2 * k - 1
    return 2.0 * 6 * np_ ** 4 / k ** 3


def flops_matvec(d, k):
    """canonical matvec flop/DoF (M/L rows k+2 nonzeros, B bulk k+2 plus the rank-2 face
    part 4(2k+1)/k)."""
    f = 4 * (2 * k + 1) / k
    return 2.0 * (4 * (k + 2) + 2 * ((k + 2) + f)) if d == 2 else 2.0 * (9 * (k + 2) + 3 * ((k + 2) + f))


def flops_fdm(d, k):
    """2 * 2d (2k-1)^(d+1) / k^d flop/DoF."""
    return 2.0 * 2 * d * (2 * k - 1) ** (d + 1) / k ** d


def sec8d_bounds(d, k, hbm_gbs, fp64_tflops):
    """SURVEY.md §8(d) attainable FP64 rates (GDoF/s) recomputed with the measured peaks: matvec (16 B/DoF),
    fused AVS step (24 B/DoF, matvec + FDM flops), MVS step (U matvec + FDM flops, U = 3.2 (2D) / 4.4 (3D);
    105 / 177 B/DoF)."""
    mv, fdm = flops_matvec(d, k), flops_fdm(d, k)
    U, mb = (3.2, 105.0) if d == 2 else (4.4, 177.0)
    g = lambda byt, fl: min(hbm_gbs / byt, fp64_tflops * 1e3 / fl)
    return {"matvec": g(16.0, mv), "avs": g(24.0, mv + fdm), "mvs": g(mb, U * mv + fdm)}


def flops_fdm_2d(k):
    """per patch 2d (2k-1)^(d+1) MACs (S^T and S along each axis), k^-d patches per DoF."""
    np_ = 2 * k - 1
    return 2.0 * 4 * np_ ** 3 / k ** 2


_NVML_SAMPLER = r"""
import sys, time, pynvml as nv
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(int(sys.argv[1]))
mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
print("ready", mx, flush=True)
bits = [nv.nvmlClocksThrottleReasonHwSlowdown, nv.nvmlClocksThrottleReasonHwThermalSlowdown,
        nv.nvmlClocksThrottleReasonSwThermalSlowdown, nv.nvmlClocksThrottleReasonSwPowerCap]
t_end = time.time() + float(sys.argv[2])
while time.time() < t_end:
    sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
    rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
    print(sm, *[int(bool(rs & b)) for b in bits], flush=True)
    time.sleep(0.002)
"""


class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled DURING the timed region by a separate
    process polling NVML every ~2 ms (no GIL contention with the launching thread); nvidia-smi
    fallback every 0.2 s."""
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index, max_seconds=120.0):
        self.idx = device_index
        self.max_seconds = max_seconds
        self.samples = []           # (sm_mhz, max_mhz, set of reason names)
        self.source = "nvml"
        self.proc = None
        self.mx = 0.0
        self._stop = threading.Event()
        self._t = None

    def _run_smi(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    f = [x.strip() for x in out.split(",")]
                    if f[1].replace(".", "").isdigit():
                        self.samples.append((float(f[1]), float(f[2]) if f[2].replace(".", "").isdigit() else 0.0,
                                             {n for n, v in zip(self.NAMES, f[5:9]) if v.lower() == "active"}))
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen([sys.executable, "-c", _NVML_SAMPLER, str(self.idx), str(self.max_seconds)],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            first = self.proc.stdout.readline().split()
            if not first or first[0] != "ready":
                raise RuntimeError("nvml sampler did not start")
            self.mx = float(first[1])
        except Exception:
            if self.proc:
                self.proc.kill()
            self.proc = None
            self.source = "nvidia-smi"
            self._t = threading.Thread(target=self._run_smi, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=10)
            except Exception:
                self.proc.kill()
                out = ""
            for line in out.splitlines():
                f = line.split()
                if len(f) == 5 and f[0].isdigit():
                    self.samples.append((float(f[0]), self.mx, {n for n, v in zip(self.NAMES, f[1:]) if v == "1"}))
        else:
            self._stop.set()
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [x[0] for x in self.samples]
        mx = [x[1] for x in self.samples]
        reasons = set().union(*[x[2] for x in self.samples])
        return {"sm_mhz": statistics.median(sm), "sm_min_mhz": min(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(self.samples), "source": self.source}


def ramp_until(fn, seconds):
    """Repeat the (already warmed-up) step for `seconds` of wall time so that the timed region starts
    at the GPU's working clock rather than its idle clock (untimed)."""
    import torch
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds:
        for _ in range(8):
            fn()
        torch.cuda.synchronize()


def dist_setup(args):
    """One process per GPU over NCCL.  Test knobs (never used for bench numbers): C0IP_BENCH_BACKEND=gloo and
    C0IP_BENCH_ONE_GPU=1 run every rank on cuda:0 with host-staged halos (exercises the N > 1 code path on a
    one-GPU box)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if os.environ.get("C0IP_BENCH_ONE_GPU"):
        local = 0
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("C0IP_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(v, world):
    if world == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cpu" if dist.get_backend() == "gloo" else "cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_oracle_sample(k, seconds_target=15.0, d=2, full=True):
    """Time the CPU oracle (as it stands) on an oracle-size twin of the workload (same d and k; 2D ~0.26M
    DoFs, 3D ~0.03-0.1M DoFs; SURVEY.md §8d / BASELINE.md "CPU baseline plan", scaled down so the whole
    sample stays within ~30 s of CPU time): the headline value is one AVS step (CSR residual + dense
    surrogate patch solves), beside it SpMV y = A x, one MVS step and (full=True) an MG-PCG solve to 1e-8
    (FP64 cycle) on the nested twin mesh.  Assembly excluded from every timing."""
    import numpy as np
    from oracle.operator import assemble, paper_rhs
    from oracle.smoothers import PatchSolvers, avs_step, mvs_step
    from oracle.discretization import default_sigma
    from oracle.multigrid import Hierarchy, pcg, precondition, default_omega
    N = ({2: 256, 3: 170, 4: 128, 5: 102, 6: 85, 7: 73} if d == 2 else {2: 20, 3: 14, 4: 10, 5: 8})[k]
    omega = default_omega(d, "avs")
    s = default_sigma(k)
    A = assemble(k, d, N, s)
    ps = PatchSolvers(k, d, N, s)
    x, b = random_xb(k, d, N)
    ndofs = len(x)

    def rate(fn, budget):
        reps, tot = 0, 0.0
        while tot < budget and reps < 50:
            t0 = time.perf_counter()
            fn()
            tot += time.perf_counter() - t0
            reps += 1
        return ndofs * reps / tot / 1e9, reps, tot
    v_avs, r_avs, t_avs = rate(lambda: avs_step(A, ps, x, b, omega), seconds_target * 0.5)
    v_mv, r_mv, t_mv = rate(lambda: A @ x, 2.0)
    v_mvs, r_mvs, t_mvs = rate(lambda: mvs_step(A, ps, x, b, default_omega(d, "mvs")), seconds_target * 0.3)
    try:
        from threadpoolctl import threadpool_info
        cores = max([p.get("num_threads", 1) for p in threadpool_info()] + [1])
    except Exception:
        cores = os.cpu_count()
    out = {"value": v_avs, "unit": "GDoF/s", "cores": cores, "kind": "oracle",
           "sample": f"{d}D k={k} N={N} ({ndofs} DoFs): {r_avs} AVS step(s) in {t_avs:.1f}s, CSR assembly excluded",
           "host_cpus": os.cpu_count(),
           "items": {"avs_step_gdofs": round(v_avs, 6), "spmv_gdofs": round(v_mv, 6), "spmv_cores": 1,
                     "mvs_step_gdofs": round(v_mvs, 6)}}
    if full:
        Lp = {2: {2: 8, 3: 7, 4: 7, 5: 6, 6: 6, 7: 6}, 3: {2: 4, 3: 3, 4: 3, 5: 3}}[d][k]
        h = Hierarchy(k, d, Lp, s)
        bb = paper_rhs(k, d, 2 ** Lp, s)
        t0 = time.perf_counter()
        _, n, hist = pcg(h.A[Lp], bb, lambda r: precondition(h, r, "avs", 2, omega))
        tp = time.perf_counter() - t0
        out["items"]["mg_pcg"] = {"dofs": int(h.A[Lp].shape[0]), "level": Lp, "iterations": int(n),
                                  "seconds": round(tp, 3), "solved_gdofs": round(h.A[Lp].shape[0] / tp / 1e9, 7),
                                  "config": "AVS 2+2 steps, CG rtol 1e-8, FP64 cycle, paper load + boundary data"}
    return out


def main_smoother(d, k, dtype):
    """The AVS realisation bench.py times (the faster one for this d, k, dtype; see main())."""
    return "avs_atomic" if (d == 3 or (dtype == "f64" and k == 4)) else "avs"


def arm_config(d, k, dtype, world=1):
    """The workload config of the timed step (shared by both arms of the bench)."""
    N = CFG2_CELLS[k] if d == 2 else CFG4_CELLS[k]
    n = k * N - 1
    ndofs = n ** d
    esz = 8 if dtype == "f64" else 4
    sm = main_smoother(d, k, dtype)
    kind = "atomic" if sm == "avs_atomic" else "deterministic gather"
    return {"workload": (f"cfg2: 2D unit square, Q{k} C0IP, N={N} cells/axis ({ndofs} DoFs), one additive "
                         f"vertex-patch smoothing step ({kind} AVS, omega=1/4)") if d == 2 else
                        (f"cfg4: 3D unit cube, Q{k} C0IP, N={N} cells/axis ({ndofs} DoFs), one additive "
                         f"vertex-patch smoothing step ({kind} AVS, omega=0.1)"),
            "degree": k, "cells": N, "dofs_per_gpu": ndofs,
            "parallelism": "replicas" if world > 1 else "single",
            "l2": "inputs larger than L2 (x, b, r = 3 x %.0f MB)" % (ndofs * esz / 1e6)}


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and rank != 0:
        return
    k = args.degree
    d = args.dim
    cb = cpu_oracle_sample(k, seconds_target=max(5.0, 20.0 / max(1, args.steps + args.warmup)), d=d, full=False)
    line = {"metric": METRIC, "value": cb["value"], "unit": "GDoF/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": arm_config(d, k, args.dtype),
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def run_slabs(args, world, rank, local):
    """Weak scaling over `world` GPUs: global mesh of N = round(N_1 world^(1/d)) cells per axis cut into
    slabs along the slowest axis (y in 2D, z in 3D); per step every rank exchanges its
    4k-2 ghost rows (planes) with its neighbours (NCCL send/recv through torch.distributed) and runs the
    slab smoothing step on its owned rows.  N_1: cfg2 (2D); cfg5 N = 128 for k = 3, cfg4 otherwise (3D)."""
    import math
    import torch
    import torch.distributed as dist
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import partition, exchange as exchange_ghosts, avs_step_overlapped
    k, d = args.degree, args.dim
    N1 = CFG2_CELLS[k] if d == 2 else (128 if k == 3 else CFG4_CELLS[k])
    N = int(round(N1 * world ** (1.0 / d)))
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    esz = 8 if dt == torch.float64 else 4
    omega = 0.25 if d == 2 else 0.1
    ctx = api.Context(d, k, 3, cells_override=N, device=local)
    L = 3
    n = k * N - 1
    row = n ** (d - 1)
    ga, _ = ctx.slab_ghosts()
    s = partition(N, k, world, ga)[rank]
    rng = torch.Generator(device="cpu").manual_seed(20241205 + rank)
    xw = (torch.rand(s.lrows * row, generator=rng, dtype=torch.float64) * 2 - 1).to("cuda", dt)
    bw = (torch.rand(s.lrows * row, generator=rng, dtype=torch.float64) * 2 - 1).to("cuda", dt)
    rw = torch.empty_like(xw)
    stream = torch.cuda.current_stream()

    def step():      # halo exchange overlapped with the interior residual (dist.avs_step_overlapped)
        avs_step_overlapped(ctx, L, omega, s, row, bw, xw, rw)

    for _ in range(max(3, args.warmup)):
        step()
    ramp_until(step, 0.5)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    lc0 = ctx.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    t_ms = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    launches = ctx.launch_count() - lc0
    own_rows = s.own_hi - s.own_lo
    total_dofs = n ** d

    # e2e: owned rows of x, b from pinned host memory each step, owned x' back
    xh = xw.view(-1, row)[s.own_local].cpu().contiguous().pin_memory()
    bh = bw.view(-1, row)[s.own_local].cpu().contiguous().pin_memory()
    oh = torch.empty_like(xh).pin_memory()

    def e2e_step():
        xw.view(-1, row)[s.own_local].copy_(xh, non_blocking=True)
        bw.view(-1, row)[s.own_local].copy_(bh, non_blocking=True)
        step()
        oh.copy_(xw.view(-1, row)[s.own_local], non_blocking=True)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(stream)
    for _ in range(args.steps):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_e2e = max_over_ranks(e0.elapsed_time(e1) / args.steps, world)
    line = {
        "metric": METRIC, "value": round(total_dofs / (t_ms * 1e-3) / 1e9, 3), "unit": "GDoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_ms, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": {"workload": (f"cfg2 weak-scaled: 2D unit square" if d == 2 else
                                 f"cfg5 weak-scaled: 3D unit cube") +
                               f", Q{k} C0IP, N={N} cells/axis ({total_dofs} DoFs, "
                               f"~{total_dofs // world} per GPU), one additive smoothing step (omega={omega}) per rank "
                               f"on a {'y' if d == 2 else 'z'}-slab with {ga} NCCL-exchanged ghost "
                               f"{'rows' if d == 2 else 'planes'} per side (exchange overlapped with the interior "
                               f"residual)",
                   "degree": k, "cells": N, "parallelism": f"slab{world}", "ghost_rows": ga,
                   "l2": "inputs larger than L2"},
        "gpu_launches": int(launches), "clocks": clk.summary(),
        "e2e": {"value": round(total_dofs / (t_e2e * 1e-3) / 1e9, 3), "unit": "GDoF/s",
                "h2d_bytes_per_step": 2 * own_rows * row * esz, "d2h_bytes_per_step": own_rows * row * esz},
    }
    # one coloured MVS step on the slabs: colours in lockstep, one ghost exchange per colour
    om_m = 0.8 if d == 2 else 0.7

    def mvs_step():
        for c in range(2 ** (d + 1)):
            exchange_ghosts(xw, s, row)
            ctx.slab_mvs_color(L, om_m, c, s.row0, s.lrows, s.own_lo, s.own_hi, bw, xw, rw)
    mvs_step()
    torch.cuda.synchronize()
    dist.barrier()
    mreps = max(2, args.steps // 4)
    e0.record(stream)
    for _ in range(mreps):
        mvs_step()
    e1.record(stream)
    torch.cuda.synchronize()
    t_mvs = max_over_ranks(e0.elapsed_time(e1) / mreps, world)
    line["mvs"] = {"value": round(total_dofs / (t_mvs * 1e-3) / 1e9, 3), "unit": "GDoF/s", "ms": round(t_mvs, 4),
                   "note": f"one coloured MVS step, {2 ** (d + 1)} colours in lockstep, omega={om_m}"}
    ctx.close()
    del xw, bw, rw
    torch.cuda.empty_cache()
    if not args.no_pcg:
        line["pcg_strong"] = dist_pcg(args, world, rank, local)
    if rank == 0:
        print(json.dumps(line))
    dist.destroy_process_group()


def dist_pcg(args, world, rank, local):
    """MG-PCG time-to-solve on slabs (strong scaling: one nested mesh for every N): DistMG (distributed levels down
    to 4 cells per rank, then an all-gathered replicated coarse cycle) + DistPCG (all-reduced dots), AVS 2+2 steps;
    device time of the whole solve, max over ranks.  2D k: L = 11 (k=2,3) / 10; 3D: L = 7 (k <= 3) / 6."""
    import torch
    import torch.distributed as dist
    from paper_2412_05082_b200 import api
    from paper_2412_05082_b200.dist import DistMG, DistPCG
    k, d = args.degree, args.dim
    Lp = ({2: 11, 3: 11, 4: 10, 5: 9, 6: 9, 7: 9} if d == 2 else {2: 7, 3: 7, 4: 6, 5: 6})[k]
    cp = api.Context(d, k, Lp, device=local)
    b = cp.rhs(Lp)
    mg = DistMG(cp, "avs", 2, 0.25 if d == 2 else 0.1, symmetric=True)
    lev = mg.levels[Lp]
    s = lev.slab
    bw = b.view(-1, lev.row)[s.row0: s.row0 + s.lrows].reshape(-1).clone()
    del b
    solver = DistPCG(mg)
    solver.solve(bw, max_iter=2)                         # warm-up
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x, n, hist = solver.solve(bw)
    e1.record()
    torch.cuda.synchronize()
    t = max_over_ranks(e0.elapsed_time(e1) * 1e-3, world)
    out = {"seconds": round(t, 4), "iterations": n, "dofs": cp.n_dofs(Lp), "level": Lp,
           "distributed_levels": sorted(mg.levels), "exchanges_per_solve": mg.exchanges,
           "solved_gdofs": round(cp.n_dofs(Lp) / t / 1e9, 4),
           "config": f"{d}D Q{k}, L={Lp}, AVS 2+2 steps, CG rtol 1e-8, FP64, {world} slabs"}
    cp.close()
    return out


def traffic_from_profiles(kernel_key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(kernel_key)
    except Exception:
        return None


def _time_ms(fn, reps, stream):
    import torch
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def sweep(d, dtype, local, degrees, clk_mhz, reps=10):
    """Degree sweep at the throughput sizes (cfg2 2D k = 2..7 / cfg4 3D k = 2..5, ~16.7M / ~50M DoFs): one
    AVS step (the timed realisation of main_smoother), the residual alone, y = A x and one coloured MVS step,
    each as GDoF/s and as a fraction of its SURVEY.md §8(d) FP64 bound (measured peaks).  Inputs are larger
    than L2 (>= 3 x 134 MB)."""
    import torch
    from paper_2412_05082_b200 import api
    hbm, _, _ = peaks()
    f64 = fp64_peak_tflops(clk_mhz)
    dt = torch.float64 if dtype == "f64" else torch.float32
    stream = torch.cuda.current_stream()
    out = {}
    for k in degrees:
        N = CFG2_CELLS[k] if d == 2 else CFG4_CELLS[k]
        ctx = api.Context(d, k, 3, cells_override=N, device=local)
        x0, b0 = random_xb(k, d, N)
        x = torch.tensor(x0, device="cuda", dtype=dt)
        b = torch.tensor(b0, device="cuda", dtype=dt)
        r = torch.empty_like(x)
        nd = ctx.n_dofs(3)
        om, om_m = (0.25, 0.8) if d == 2 else (0.1, 0.7)
        sm = main_smoother(d, k, dtype)
        for _ in range(3):
            ctx.smooth(3, sm, 1, om, b, x)
        t_avs = _time_ms(lambda: ctx.smooth(3, sm, 1, om, b, x), reps, stream)
        t_res = _time_ms(lambda: ctx.residual(3, b, x, r), reps, stream)
        t_mv = _time_ms(lambda: ctx.apply(3, x, r), reps, stream)
        t_mvs = _time_ms(lambda: ctx.smooth(3, "mvs", 1, om_m, b, x), max(2, reps // 4), stream)
        bd = sec8d_bounds(d, k, hbm, f64)
        g = lambda t: nd / (t * 1e-3) / 1e9
        out[f"k{k}"] = {"dofs": nd, "cells": N, "avs_smoother": sm,
                        "avs": round(g(t_avs), 3), "avs_frac": round(g(t_avs) / bd["avs"], 4),
                        "residual_ms": round(t_res, 4), "fdm_ms": round(t_avs - t_res, 4),
                        "matvec": round(g(t_mv), 3), "matvec_frac": round(g(t_mv) / bd["matvec"], 4),
                        "mvs": round(g(t_mvs), 3), "mvs_frac": round(g(t_mvs) / bd["mvs"], 4),
                        "bounds_gdofs": {kk: round(v, 1) for kk, v in bd.items()}}
        ctx.close()
        del x, b, r
        torch.cuda.empty_cache()
    out["note"] = (f"GDoF/s; *_frac = value / SURVEY.md §8(d) FP64 bound (HBM {hbm:.0f} GB/s, FP64 {f64:.1f} "
                   f"TFLOP/s); MVS omega {0.8 if d == 2 else 0.7}, AVS omega {0.25 if d == 2 else 0.1}")
    return out


def fig5_3d(local, reps=4):
    """PAPER.md:809-816 (Fig. 5): operator evaluation A x and one MVS step, biharmonic C0IP vs Poisson SIPG, 3D,
    64^3 cells, k = 2..5, FP64, as GDoF/s and the biharmonic / Poisson time ratio (the paper: 2-3x slower for the
    biharmonic operator on an A100).  Here the C0IP path runs the fused 3D kernels, the SIPG path the generic
    per-axis kernels (SURVEY.md f3 is a comparison workload, not tuned)."""
    import torch
    from paper_2412_05082_b200 import api
    stream = torch.cuda.current_stream()
    out = {}
    for k in (2, 3, 4, 5):
        row = {}
        for name, sipg in (("biharmonic", False), ("poisson_sipg", True)):
            ctx = api.Context(3, k, 6, device=local, sipg=sipg)
            nd = ctx.n_dofs(6)
            g = torch.Generator(device="cpu").manual_seed(20241205)
            x = (torch.rand(nd, generator=g, dtype=torch.float64) * 2 - 1).cuda()
            b = (torch.rand(nd, generator=g, dtype=torch.float64) * 2 - 1).cuda()
            y = torch.empty_like(x)
            t_mv = _time_ms(lambda: ctx.apply(6, x, y), reps, stream)
            om = 0.7 if not sipg else 1.0
            t_mvs = _time_ms(lambda: ctx.smooth(6, "mvs", 1, om, b, x), max(2, reps // 2), stream)
            row[name] = {"dofs": nd, "ax_gdofs": round(nd / (t_mv * 1e-3) / 1e9, 3), "ax_ms": round(t_mv, 4),
                         "mvs_gdofs": round(nd / (t_mvs * 1e-3) / 1e9, 3), "mvs_ms": round(t_mvs, 4)}
            ctx.close()
            del x, b, y
            torch.cuda.empty_cache()
        row["biharmonic_over_poisson_time_per_dof"] = {
            "ax": round(row["poisson_sipg"]["ax_gdofs"] / row["biharmonic"]["ax_gdofs"], 3),
            "mvs": round(row["poisson_sipg"]["mvs_gdofs"] / row["biharmonic"]["mvs_gdofs"], 3)}
        out[f"k{k}"] = row
    out["config"] = "3D unit cube, 64^3 cells (level 6), FP64; MVS omega 0.7 (C0IP) / 1 (SIPG, exact FDM)"
    return out


def mixed_3d(local):
    """The paper's mixed-precision experiment (Fig. 4): 3D, GMRES preconditioned by the
    V-cycle with one MVS step (omega 0.7, same-order cycle), FP64 cycle vs FP32 cycle (outer FGMRES(30) in FP64),
    rtol 1e-8, F = c0ip_rhs, on the largest nested meshes of cfg4 (k = 2, 3: N = 128; k = 4: N = 64)."""
    import torch
    from paper_2412_05082_b200 import api
    out = {}
    for k, Lm in ((2, 7), (3, 7), (4, 6)):
        cm = api.Context(3, k, Lm, device=local)
        bm = cm.rhs(Lm)
        r = {}
        for name, cdt in (("fp64", torch.float64), ("mixed", torch.float32)):
            mg = api.MG("mvs", 1, 0.7, symmetric=False, cycle_dtype=cdt)
            cm.gmres(mg, bm, max_iter=2, restart=30)
            torch.cuda.synchronize()
            xs, rep, hist = cm.gmres(mg, bm, max_iter=60, restart=30)
            r[name] = {"seconds": round(rep["seconds"], 4), "iterations": rep["iterations"],
                       "nu": round(rep["nu"], 2), "converged": rep["converged"],
                       "solved_mdofs_per_s": round(cm.n_dofs(Lm) / rep["seconds"] / 1e6, 1)}
        r["dofs"] = cm.n_dofs(Lm)
        r["mixed_speedup"] = round(r["fp64"]["seconds"] / r["mixed"]["seconds"], 3)
        out[f"k{k}_L{Lm}"] = r
        cm.close()
        del bm
        torch.cuda.empty_cache()
    out["config"] = ("3D unit cube, MVS 1+1 step omega=0.7 (16 colours, same order), FGMRES(30) rtol 1e-8, x0=0, "
                     "paper load + Nitsche boundary data; FP32 cycle = every level and table in FP32, conversion at "
                     "the cycle's entry and exit (PAPER.md:749)")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--degree", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-pcg", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--dim", type=int, default=2, choices=[2, 3])
    ap.add_argument("--no-sweep", action="store_true", help="skip the 2D/3D degree sweeps")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import numpy as np
    import torch
    world, rank, local = dist_setup(args)
    torch.cuda.set_device(local)
    from paper_2412_05082_b200 import api

    k = args.degree
    if world > 1:
        return run_slabs(args, world, rank, local)
    d = args.dim
    N = CFG2_CELLS[k] if d == 2 else CFG4_CELLS[k]
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    ctx = api.Context(d, k, 3, cells_override=N, device=local)
    L = 3
    ndofs = ctx.n_dofs(L)
    x0, b0 = random_xb(k, d, N)
    x = torch.tensor(x0, device="cuda", dtype=dt)
    b = torch.tensor(b0, device="cuda", dtype=dt)
    r = torch.empty_like(x)
    stream = torch.cuda.current_stream()
    omega = 0.25 if d == 2 else 0.1

    # the timed step is the faster of the two AVS realisations for this (d, k, dtype): the paper's atomic
    # AVS (residual, then every patch solve scatter-added with fire-and-forget atomics; 2D FP64
    # k = 4 on the DMMA patch kernel, 3D) or the deterministic gather AVS (2D otherwise); the other one is
    # reported beside it
    main_sm = main_smoother(d, k, args.dtype)
    other_sm = "avs" if main_sm == "avs_atomic" else "avs_atomic"

    def step():
        ctx.smooth(L, main_sm, 1, omega, b, x)

    for _ in range(max(3, args.warmup)):
        step()
    ramp_until(step, 0.5)           # let the SM clock leave its idle state before timing
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    lc0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
        t_step_ms = ev0.elapsed_time(ev1) / args.steps
        launches = (ctx.launch_count() - lc0)
        # per-kernel timing (same stream): residual (apply2d) and FDM apply (fdm2d) separately
        for _ in range(3):
            ctx.residual(L, b, x, r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ctx.residual(L, b, x, r)
        e1.record(stream)
        torch.cuda.synchronize()
        t_res_ms = e0.elapsed_time(e1) / args.steps
        e0.record(stream)
        for _ in range(args.steps):
            ctx.apply(L, x, r)
        e1.record(stream)
        torch.cuda.synchronize()
        t_mv_ms = e0.elapsed_time(e1) / args.steps
        # one coloured multiplicative step (8 colours, residual per colour),
        # omega = 0.8 (2D, reading Q28) / 0.7 (3D)
        xm = x.clone()
        om_m = 0.8 if d == 2 else 0.7
        ctx.smooth(L, "mvs", 1, om_m, b, xm)
        mreps = max(2, args.steps // 4)
        e0.record(stream)
        for _ in range(mreps):
            ctx.smooth(L, "mvs", 1, om_m, b, xm)
        e1.record(stream)
        torch.cuda.synchronize()
        t_mvs_ms = e0.elapsed_time(e1) / mreps
        # the other AVS realisation (deterministic: gather form in 2D, parity classes in 3D)
        xa = x.clone()
        ctx.smooth(L, other_sm, 1, omega, b, xa)
        e0.record(stream)
        for _ in range(mreps):
            ctx.smooth(L, other_sm, 1, omega, b, xa)
        e1.record(stream)
        torch.cuda.synchronize()
        t_atomic_ms = e0.elapsed_time(e1) / mreps
    barrier(world)
    t_step_ms = max_over_ranks(t_step_ms, world)
    clocks = clk.summary()

    # e2e through the C ABI with host buffers (pinned), copies inside the timed region: every step copies
    # its x, b host -> device and its x' device -> host.  The copies are pipelined across steps on their
    # own streams (H2D of step i+1 and D2H of step i-1 overlap the smoothing step i; device buffers double
    # buffered), as a streaming user of the library would run it; the timed region spans the first H2D
    # to the last D2H.
    xh = torch.tensor(x0, dtype=dt).pin_memory()
    bh = torch.tensor(b0, dtype=dt).pin_memory()
    outh = [torch.empty_like(xh).pin_memory() for _ in range(2)]
    xd = [torch.empty_like(x) for _ in range(2)]
    bd = [torch.empty_like(b) for _ in range(2)]
    s_h2d, s_comp, s_d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

    def e2e_run(nsteps, ev_start=None, ev_end=None):
        h2d_done = [torch.cuda.Event() for _ in range(nsteps)]
        comp_done = [torch.cuda.Event() for _ in range(nsteps)]
        d2h_done = [torch.cuda.Event() for _ in range(nsteps)]
        if ev_start is not None:
            ev_start.record(s_h2d)
        for i in range(nsteps):
            j = i % 2
            with torch.cuda.stream(s_h2d):
                if i >= 2:
                    s_h2d.wait_event(d2h_done[i - 2])        # buffer j free again
                xd[j].copy_(xh, non_blocking=True)
                bd[j].copy_(bh, non_blocking=True)
                h2d_done[i].record(s_h2d)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(h2d_done[i])
                ctx.smooth(L, main_sm, 1, omega, bd[j], xd[j])
                comp_done[i].record(s_comp)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(comp_done[i])
                outh[j].copy_(xd[j], non_blocking=True)
                d2h_done[i].record(s_d2h)
        if ev_end is not None:
            ev_end.record(s_d2h)

    e2e_run(3)
    torch.cuda.synchronize()
    barrier(world)
    es, ee = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2e_run(args.steps, es, ee)
    torch.cuda.synchronize()
    t_e2e_ms = max_over_ranks(es.elapsed_time(ee) / args.steps, world)

    esz = 8 if dt == torch.float64 else 4
    hbm, mhz, peak_src = peaks()
    clk_mhz = clocks.get("sm_mhz") or mhz
    t_fdm_ms = max(t_step_ms - t_res_ms, 1e-9)
    # dominant kernel of the step and its roofline (algorithmic work / live CUDA-event time)
    if d == 2:
        fdm_name = (("patch_fdm2d_mma" if not os.environ.get("C0IP_NO_MMA") else "patch_fdm")
                    if main_sm == "avs_atomic" else ("fdm2d_mma" if (k == 4 and args.dtype == "f64") else "fdm2d"))
        kern = fdm_name if t_fdm_ms >= t_res_ms else "apply2d"
        flop = (flops_fdm_2d(k) if kern != "apply2d" else flops_residual_2d(k)) * ndofs
    else:
        kern = "patch_fdm3d" if t_fdm_ms >= t_res_ms else "apply3d"
        flop = (flops_fdm_3d(k) if kern == "patch_fdm3d" else flops_residual_3d(k)) * ndofs
    t_k = t_fdm_ms if kern != "apply2d" and kern != "apply3d" else t_res_ms
    byts = 3 * esz * ndofs
    peak_alu = fp64_peak_tflops(clk_mhz) if esz == 8 else fp32_peak_tflops(clk_mhz)
    ach_tf = flop / (t_k * 1e-3) / 1e12
    ach_gb = byts / (t_k * 1e-3) / 1e9
    f_alu, f_hbm = ach_tf / peak_alu, ach_gb / hbm
    if f_alu >= f_hbm:
        roof = {"bound": "alu", "achieved": round(ach_tf, 3), "peak": round(peak_alu, 2), "unit": "TFLOP/s",
                "frac": round(f_alu, 4)}
        alt = {"bound": "hbm", "achieved": round(ach_gb, 1), "peak": hbm, "unit": "GB/s", "frac": round(f_hbm, 4)}
    else:
        roof = {"bound": "hbm", "achieved": round(ach_gb, 1), "peak": hbm, "unit": "GB/s", "frac": round(f_hbm, 4)}
        alt = {"bound": "alu", "achieved": round(ach_tf, 3), "peak": round(peak_alu, 2), "unit": "TFLOP/s",
               "frac": round(f_alu, 4)}
    roof["kernel"] = kern
    roof["traffic"] = traffic_from_profiles(f"{kern}_kernel_k{k}_{args.dtype}")
    roof["peak_source"] = (f"hbm {peak_src} (MEASURED_PEAKS.json); alu " +
                           ("measured (profiles/alu_peaks.json, tools/alu_peaks.cu)" if _alu_peaks() else
                            f"derived 148x{64 if esz == 8 else 128}x2 flop/clk") + f" rescaled to {clk_mhz:.0f} MHz")
    roof["alt"] = alt
    roof["launch_ms"] = round(t_k, 4)

    value = ndofs * world / (t_step_ms * 1e-3) / 1e9
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GDoF/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(t_step_ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": arm_config(d, k, args.dtype, world),
        "gpu_launches": int(launches),
        "clocks": clocks,
        "e2e": {"value": round(ndofs * world / (t_e2e_ms * 1e-3) / 1e9, 3), "unit": "GDoF/s",
                "h2d_bytes_per_step": 2 * ndofs * esz, "d2h_bytes_per_step": ndofs * esz},
        "roofline": roof,
        "matvec": {"value": round(ndofs * world / (t_mv_ms * 1e-3) / 1e9, 3), "unit": "GDoF/s",
                   "ms": round(t_mv_ms, 4)},
        "mvs": {"value": round(ndofs * world / (t_mvs_ms * 1e-3) / 1e9, 3), "unit": "GDoF/s",
                "ms": round(t_mvs_ms, 4),
                "note": f"one coloured MVS step, {2 ** (d + 1)} colours, omega={om_m}"},
        ("avs_deterministic" if other_sm == "avs" else "avs_atomic"):
            {"value": round(ndofs * world / (t_atomic_ms * 1e-3) / 1e9, 3), "unit": "GDoF/s", "ms": round(t_atomic_ms, 4)},
        "residual_ms": round(t_res_ms, 4), "fdm_ms": round(t_fdm_ms, 4),
    }

    if not args.no_pcg:
        # MG-PCG time-to-solve on the nested mesh N = 2^L of similar size
        Lp = ({2: 11, 3: 10, 4: 10, 5: 9, 6: 9, 7: 9} if d == 2 else {2: 7, 3: 7, 4: 6, 5: 6})[k]
        ctx.close()
        cp = api.Context(d, k, Lp, device=local)
        bb = cp.rhs(Lp)
        res = {}
        for name, cdt in (("fp64", torch.float64), ("mixed", torch.float32)):
            mg = api.MG("avs", 2, 0.25 if d == 2 else 0.1, cycle_dtype=cdt)
            cp.pcg(mg, bb, max_iter=3)            # warm-up (allocations, first launches)
            torch.cuda.synchronize()
            xs, rep, hist = cp.pcg(mg, bb)
            res[name] = {"seconds": round(rep["seconds"], 4), "iterations": rep["iterations"],
                         "nu": round(rep["nu"], 2), "converged": rep["converged"]}
        res["dofs"] = cp.n_dofs(Lp)
        res["config"] = (f"{d}D Q{k}, L={Lp} (N={2 ** Lp}), AVS 2+2 steps omega={0.25 if d == 2 else 0.1}, "
                         f"CG rtol 1e-8, x0=0, paper load + Nitsche boundary data")
        res["mixed_speedup"] = round(res["fp64"]["seconds"] / res["mixed"]["seconds"], 3)
        line["pcg"] = res
        cp.close()
        if d == 2:
            # the largest 2D level at which the FP32 cycle keeps the FP64 iteration count within 1 (DESIGN.md §8:
            # u32 kappa(A) grows like h^-4; 2D k=4: L = 9)
            Lh = Lp - 1
            ch = api.Context(d, k, Lh, device=local)
            bh = ch.rhs(Lh)
            rh = {}
            for name, cdt in (("fp64", torch.float64), ("mixed", torch.float32)):
                mg = api.MG("avs", 2, 0.25, cycle_dtype=cdt)
                ch.pcg(mg, bh, max_iter=3)
                torch.cuda.synchronize()
                xs, rep, hist = ch.pcg(mg, bh)
                rh[name] = {"seconds": round(rep["seconds"], 4), "iterations": rep["iterations"],
                            "nu": round(rep["nu"], 2), "converged": rep["converged"]}
            rh["dofs"] = ch.n_dofs(Lh)
            rh["level"] = Lh
            rh["mixed_speedup"] = round(rh["fp64"]["seconds"] / rh["mixed"]["seconds"], 3)
            line["pcg_mixed_holds"] = rh
            ch.close()
        if (d == 2 and k == 4) or d == 3:
            # cfg3 (BASELINE.json configs[2]): coloured multiplicative smoother, k = 4, N = 2048 (67.1M DoFs),
            # one MVS step (omega = 0.8, reading Q28) with the symmetric colour order (Q11), FP32 vs
            # FP64 cycle; 3D (cfg4, the paper's Fig. 4 setting): MVS omega = 0.7, N = 2^Lp
            Lm = 11 if d == 2 else Lp
            om_m = 0.8 if d == 2 else 0.7
            cm = api.Context(d, k, Lm, device=local)
            bm = cm.rhs(Lm)
            rm = {}
            for name, cdt in (("fp64", torch.float64), ("mixed", torch.float32)):
                mg = api.MG("mvs", 1, om_m, symmetric=True, cycle_dtype=cdt)
                cm.pcg(mg, bm, max_iter=2)
                torch.cuda.synchronize()
                xs, rep, hist = cm.pcg(mg, bm, max_iter=60)
                rm[name] = {"seconds": round(rep["seconds"], 4), "iterations": rep["iterations"],
                            "nu": round(rep["nu"], 2), "converged": rep["converged"]}
            rm["dofs"] = cm.n_dofs(Lm)
            rm["config"] = ((f"cfg3: 2D Q4, L=11 (N=2048), MVS 1+1 step omega=0.8 (8 colours" if d == 2 else
                             f"cfg4: 3D Q{k}, L={Lm} (N={2 ** Lm}), MVS 1+1 step omega=0.7 (16 colours") +
                            ", reversed order in post-smoothing), CG rtol 1e-8 (max 60 iterations), x0=0, paper load + Nitsche boundary data")
            rm["mixed_speedup"] = round(rm["fp64"]["seconds"] / rm["mixed"]["seconds"], 3)
            line["pcg_mvs"] = rm
            # the paper's MVS protocol: GMRES around the same-order
            # (nonsymmetric) MVS V-cycle, FP64 vs FP32 cycle
            rg = {}
            for name, cdt in (("fp64", torch.float64), ("mixed", torch.float32)):
                mg = api.MG("mvs", 1, om_m, symmetric=False, cycle_dtype=cdt)
                cm.gmres(mg, bm, max_iter=2, restart=30)      # warm-up: workspace, V-cycle graph
                torch.cuda.synchronize()
                xs, rep, hist = cm.gmres(mg, bm, max_iter=60, restart=30)
                rg[name] = {"seconds": round(rep["seconds"], 4), "iterations": rep["iterations"],
                            "nu": round(rep["nu"], 2), "converged": rep["converged"]}
            rg["dofs"] = rm["dofs"]
            rg["config"] = rm["config"].replace("CG", "FGMRES(30)").replace("reversed order in post-smoothing",
                                                                          "same order in post-smoothing")
            rg["mixed_speedup"] = round(rg["fp64"]["seconds"] / rg["mixed"]["seconds"], 3)
            line["gmres_mvs"] = rg
            cm.close()
    else:
        ctx.close()

    if not args.no_pcg and world == 1 and d == 2:
        line["mixed_3d"] = mixed_3d(local)
    if not args.no_sweep and world == 1 and d == 2:
        line["fig5_3d"] = fig5_3d(local)
    if not args.no_sweep and world == 1:
        line["sweep_2d"] = sweep(2, args.dtype, local, range(2, 8), clk_mhz)
        line["sweep_3d_cfg4"] = sweep(3, args.dtype, local, range(2, 6), clk_mhz, reps=4)
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_oracle_sample(k, d=d)
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
