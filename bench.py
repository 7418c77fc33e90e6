#!/usr/bin/env python
"""Benchmark of the w-product hot path on B200 (contract: DESIGN.md section 7).

Headline (BASELINE.json metric "w-svd rank-k reconstruct tensor-elems/s ...
1/2/4/8 GPU", configs[3]): ``sp_w_svd`` rank-30 reconstruction of the
1024x1024x256 float64 hyperspectral cube at L = 4.  One step = one call on the
device-resident cube (2 GiB in, 2 GiB out: larger than L2); value = tensor
elements reconstructed per second.  N > 1 (torchrun, one rank per GPU): the
same cube, rows sharded over the ranks (strong scaling); K1 stores the coarse
wavelet slices straight into the owning GPU's buffer, K4 decomposes them there
and K2 loads the reconstructed rows back (``sharded.sp_w_svd_fused``).

Secondary keys of the same line: ``transform`` (BASELINE configs[1], lifting
round trips at L = 1, 2, 4, 8, HBM GB/s) and, at N = 1, ``workloads`` for
configs 1, 3 and 5, each with a same-run CPU baseline (the multi-threaded
oracle port, full size, median of 3) and the roofline of its dominant kernel.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workloads wsvd,deblur,wproduct,comparators | none]

``--impl reference`` times the reference algorithm on the host cores (the
oracle port, ``oracle/parallel.py``: numpy + LAPACK dgesdd, all host threads)
on the same workload, metric and config.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "w-svd rank-k reconstruct tensor-elems/s"
UNIT = "tensor-elems/s"
CFG4 = (1024, 1024, 256)
CFG4_RANK, CFG4_LEVELS = 30, 4
CFG2 = (512, 512, 256)
CFG2_LEVELS = (1, 2, 4, 8)
DATA = ("synthetic: seeded hyperspectral cube (paper_2601_08228_b200/synth.py, BASELINE configs[2-4] "
        "generator; the paper's datasets are not available); i.i.d. normal cube for the transform key")


def headline_config():
    """Identical in both arms (the driver compares them)."""
    n1, n2, p = CFG4
    return {"workload": f"sp_w_svd rank-{CFG4_RANK} reconstruction of the {n1}x{n2}x{p} f64 hyperspectral "
                        f"cube, L={CFG4_LEVELS} (BASELINE configs[3]); one call per step",
            "cube": list(CFG4), "rank": CFG4_RANK, "levels": CFG4_LEVELS,
            "generator": "synth.hyperspectral_cube(1024, 1024, 256, seed=0): 10 endmembers, Dirichlet(0.5) "
                         "abundances smoothed sigma=4 px, 3-bump spectra, noise 0.01, clipped to [0, 1]",
            "l2": "2 GiB input and 2 GiB output per step, larger than the 126 MB L2"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workloads", default="default")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--force-dist", action="store_true",
                    help="initialise NCCL even at world size 1 (exercises the N>1 code path on one GPU)")
    return ap.parse_args()


# ------------------------------------------------------------------ env ----

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def fp64_peak():
    """DMMA FP64 peak measured on this pool (tools/fp64_peak.cu -> profiles/fp64_peak_r01.jsonl);
    MEASURED_PEAKS.json has no FP64 entry."""
    path = os.path.join(ROOT, "profiles", "fp64_peak_r01.jsonl")
    try:
        best = 0.0
        for line in open(path):
            d = json.loads(line)
            if d.get("kind") == "dmma_m8n8k4":
                best = max(best, float(d["tflops"]))
        if best > 0:
            return best, "measured (tools/fp64_peak.cu DMMA m8n8k4, profiles/fp64_peak_r01.jsonl)"
    except Exception:  # noqa: BLE001
        pass
    return 37.0, "fallback (B200 FP64 tensor, measured 36.99 TF in round 1)"


def executed_k4_rate(n1, n2, nslices, k4_ms, peak):
    """FP64 flops the leading-triplet K4 call executes (two-stage path, DESIGN.md 4.3 item 3b) per slice:
    Gram lower tiles m n^2, trailing passes 72 flops per trailing-block element per 12-column panel
    (rank-24 update + block x V), panel QR / pending update / W ~ 10 m b per row and panel, band chase 6 b n^2,
    stage-2 back-transform 2 n^2 k, stage-1 back-transform (compact-WY blocks of 128) ~ 4 n^2 k + n^2 128,
    Newton-Schulz 4 n k^2, X V0 2 m n k -- against the measured DMMA peak: the honest utilisation next to
    the effective rate on the reference's count."""
    m, n = max(n1, n2), min(n1, n2)
    b, k = 12, 64
    trailing = sum(72 * (n - b * (j + 1)) ** 2 for j in range((n - b - 2) // b + 1) if n - b * (j + 1) >= 2)
    small = sum(10 * 2 * b * b * max(n - b * (j + 1), 0) for j in range(n // b + 1))
    flops = nslices * (m * n * n + trailing + small + 6 * b * n * n + 2 * n * n * k + 4 * n * n * k + 128 * n * n
                       + 4 * n * k * k + 2 * m * n * k)
    ach = flops / (k4_ms * 1e-3) / 1e12
    return {"flops_per_call": int(flops), "achieved": round(ach, 3), "unit": "TFLOP/s", "frac": round(ach / peak, 4),
            "note": "executed flops of the two-stage leading-triplet path (model in bench.executed_k4_rate); the "
                    "call is latency-bound in the band chase (2 n sequential hops) and panel QR, DMMA-bound at 57% "
                    "pipe-active in the trailing passes (profiles/r02_summary.md)"}


def profile_value(name, key):
    """Per-launch DRAM traffic etc. recorded from an ncu capture (profiles/traffic_r02.json)."""
    for fn in ("traffic_r02.json", "traffic_r01.json"):
        try:
            v = json.load(open(os.path.join(ROOT, "profiles", fn))).get(name)
        except Exception:  # noqa: BLE001
            continue
        if v is not None:
            return v.get(key) if isinstance(v, dict) else v
    return None


def host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


class ClockSampler:
    """Samples SM clocks and throttle reasons via NVML during the timed region."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = 0
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons |= int(r) & ~0x1
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t is not None:
            self._t.join()

    def summary(self):
        if self.nv is None or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples),
                "reasons": [n for b, n in self.REASONS.items() if self.reasons & b]}


# --------------------------------------------------------------- timing ----

def timed_region(step_fn, steps, warmup, dist=None, sampler=None):
    """W warm-up steps, then exactly K steps bracketed by barrier + synchronize;
    returns the max over ranks of the device time (ms) of the K steps."""
    import torch

    for _ in range(warmup):
        step_fn(False)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    ctx = sampler if sampler is not None else _Null()
    with ctx:
        t0.record()
        for _ in range(steps):
            step_fn(True)
        t1.record()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ms = t0.elapsed_time(t1)
    if dist is not None:
        v = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(v, op=dist.ReduceOp.MAX)
        ms = float(v.item())
    return ms


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


class PhaseTimer:
    """CUDA events around every call of selected engine entry points (K4 = E.svd,
    K3 = E.gemm), recorded on the stream they launch on (torch's current stream)
    while `on` is set; mean device ms per call of each."""

    def __init__(self, names=("svd", "svd_topk", "gemm")):
        from paper_2601_08228_b200 import engine as E

        self.E = E
        self.names = names
        self.pairs = {n: [] for n in names}
        self.on = False
        self._orig = {}

    def __enter__(self):
        import torch

        for n in self.names:
            orig = getattr(self.E, n)
            self._orig[n] = orig

            def wrapped(*a, _orig=orig, _n=n, **k):
                if not self.on:
                    return _orig(*a, **k)
                s = torch.cuda.Event(enable_timing=True)
                e = torch.cuda.Event(enable_timing=True)
                s.record()
                out = _orig(*a, **k)
                e.record()
                self.pairs[_n].append((s, e))
                return out

            setattr(self.E, n, wrapped)
        return self

    def __exit__(self, *exc):
        for n, f in self._orig.items():
            setattr(self.E, n, f)
        return False

    def total_ms(self, name):
        return sum(s.elapsed_time(e) for s, e in self.pairs[name])

    def calls(self, name):
        return len(self.pairs[name])


def count_launches(fn):
    """Kernels of the repo's own library launched by one call of fn (CUPTI via
    torch.profiler; torch / NCCL / library kernels excluded).  Returns (count, names)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    names = {}
    foreign = ("at::", "nccl", "cublas", "cutlass", "xmma", "Memcpy", "Memset", "cudnn", "triton", "c10::",
               "elementwise_kernel", "reduce_kernel")
    for ev in prof.events():
        if getattr(ev, "device_type", None) is None or "CUDA" not in str(ev.device_type):
            continue
        nm = ev.name
        if any(f in nm for f in foreign):
            continue
        names[nm] = names.get(nm, 0) + 1
    return sum(names.values()), names


# ------------------------------------------------------------ CPU legs ----

def cpu_median(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t)
    return statistics.median(ts), ts


def cpu_port_baseline(fn, unit_value, unit, sample, reps=3):
    """Same-run CPU baseline: the oracle port (oracle/parallel.py) on the FULL
    workload, all host threads, 1 warm-up + median of `reps` calls."""
    from oracle import parallel as P

    with P.Pool() as pool:
        med, ts = cpu_median(lambda: fn(pool), reps)
        threads = pool.threads
    return {"value": unit_value(med), "unit": unit, "cores": threads, "kind": "port",
            "ms_per_call": round(med * 1e3, 1), "calls_s": [round(t, 3) for t in ts],
            "sample": f"{sample}; full size, 1 warm-up + median of {reps} calls, numpy + LAPACK dgesdd / "
                      f"BLAS dgemm (oracle/parallel.py) over {threads} host threads"}


# ------------------------------------------------------------ headline ----

def cfg4_cube(rank=0):
    from paper_2601_08228_b200 import synth

    n1, n2, p = CFG4
    return synth.hyperspectral_cube(n1, n2, p, seed=0)


def svd_flops(n1, n2):
    """Golub-Kahan thin-SVD count: 14 m n^2 + 8 n^3, m >= n."""
    m, n = max(n1, n2), min(n1, n2)
    return 14 * m * n * n + 8 * n ** 3


def headline_single(args, x_host, sampler):
    import torch

    from paper_2601_08228_b200 import engine as E
    import paper_2601_08228_b200 as W
    from paper_2601_08228_b200.decomposition import sp_w_svd_device

    n1, n2, p = CFG4
    r, L = CFG4_RANK, CFG4_LEVELS
    N = n1 * n2 * p
    x = torch.from_numpy(x_host).cuda()
    out = torch.empty_like(x)
    info = {}
    with PhaseTimer() as pt:
        def step(record):
            pt.on = record
            sp_w_svd_device(x, r, L, out=out)
            if record:
                info["sweeps"] = E.last_sweeps()
                info["jflops"] = E.last_jacobi_flops()

        ms = timed_region(step, args.steps, args.warmup, None, sampler)
        k4_name = "svd_topk" if pt.calls("svd_topk") else "svd"
        k4_ms = pt.total_ms(k4_name) / max(pt.calls(k4_name), 1)
        k3_ms = pt.total_ms("gemm") / max(pt.calls("gemm"), 1) if pt.calls("gemm") else None
    per_call = ms / args.steps
    peak, src = fp64_peak()
    flops = 2 * (p >> L) * svd_flops(n1, n2)
    ach = flops / (k4_ms * 1e-3) / 1e12
    roofline = {"bound": "tensor", "kernel": f"K4 {'wt_svd_topk_f64 (64 leading triplets)' if k4_name == 'svd_topk' else 'wt_svd_jacobi_f64'}"
                                              " on the 32 coarse 1024^2 slices: every launch of one call "
                                              "(Gram, two-stage tridiagonalization: band panels + trailing passes + band "
                                              "chase, bisection, inverse iteration, Newton-Schulz, back-transforms, X V0, "
                                              "Jacobi sweeps, sort)",
                "achieved": round(ach, 3), "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "peak_source": src,
                "traffic": profile_value("K4_cfg4t" if k4_name == "svd_topk" else "K4_cfg4", "dram_bytes_per_call"),
                "flops_per_launch": flops,
                "flops_model": "32 x (14 m n^2 + 8 n^3), m = n = 1024: the Golub-Kahan thin-SVD count of the work the "
                               "reference does for this result (SURVEY 8(d)); the leading-triplet mode executes less "
                               "(DESIGN.md 4.3), so frac is an effective rate on the reference's count",
                "executed": executed_k4_rate(n1, n2, 2 * (p >> L), k4_ms, peak) if k4_name == "svd_topk" else None,
                "k4_ms_per_call": round(k4_ms, 3), "share_of_step": round(k4_ms / per_call, 4),
                "executed_jacobi_tflops": round(info["jflops"] / (k4_ms * 1e-3) / 1e12, 3),
                "jacobi_sweeps": info["sweeps"]}
    # e2e: the public API on host (numpy) arrays -- H2D of the cube and D2H of the
    # reconstruction inside every call (decomposition.sp_w_svd)
    e2e_steps = max(1, min(args.steps, 5))
    # warm-up as in the timed loop (the previous result alive while the next call
    # runs): the two calls allocate engine.host_buffer's two pooled pinned result
    # buffers (page-locking a fresh 2 GiB block costs ~0.9 s, once)
    # The input cube lives in page-locked host memory (W.pinned_empty), as the contract's e2e leg
    # prescribes: the call DMAs its row chunks in place.  The same call on an ordinary (pageable)
    # numpy array goes through the pinned staging ring and is reported beside it.
    x_pin = W.pinned_empty(x_host.shape)
    x_pin[...] = x_host

    def e2e_leg(xin):
        y = W.sp_w_svd(xin, r, L)
        y = W.sp_w_svd(xin, r, L)
        torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(e2e_steps):
            y = W.sp_w_svd(xin, r, L)
        return (time.perf_counter() - t) / e2e_steps, y

    e2e_pageable_s, y_host = e2e_leg(x_host)
    del y_host  # (its pinned result buffer goes back to the pool of two before the next leg)
    e2e_s, y_host = e2e_leg(x_pin)
    # the same calls as a stream of cubes, three in flight (W.sp_w_svd_many): every cube is still
    # uploaded and its result downloaded, the two PCIe directions and K4 of neighbouring calls overlap
    del y_host
    n_pipe = 4 * e2e_steps
    # warm-up: every result kept, so the pool page-locks all of its result buffers now (a 2 GiB
    # cudaHostAlloc costs ~0.9 s; in the timed stream below it landed in some runs and not in others)
    keep = list(W.sp_w_svd_many((x_pin for _ in range(5)), r, L))
    del keep
    torch.cuda.synchronize()
    pipe_runs = []
    for _ in range(3):  # median of three streams (a stream that meets a pool page-lock costs +0.3..0.9 s)
        t = time.perf_counter()
        for y_host in W.sp_w_svd_many((x_pin for _ in range(n_pipe)), r, L):
            pass
        pipe_runs.append((time.perf_counter() - t) / n_pipe)
    pipe_s = sorted(pipe_runs)[1]
    e2e = {"value": round(N / e2e_s, 1), "unit": UNIT, "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
           "ms_per_call": round(e2e_s * 1e3, 2), "steps": e2e_steps,
           "ms_per_call_pageable_input": round(e2e_pageable_s * 1e3, 2),
           "pipelined": {"value": round(N / pipe_s, 1), "unit": UNIT, "ms_per_cube": round(pipe_s * 1e3, 2),
                         "cubes": n_pipe, "ms_per_cube_runs": [round(v * 1e3, 2) for v in pipe_runs],
                         "api": "sp_w_svd_many(stream of page-locked numpy cubes, 30, 4): three "
                         "calls in flight, every cube uploaded and every result downloaded; median of three "
                         "streams"},
           "api": "sp_w_svd(numpy cube in page-locked memory, 30, 4) -> numpy reconstruction (H2D of the 2 GiB cube "
                  "and D2H of the 2 GiB result inside every call; ms_per_call_pageable_input: the same call on a "
                  "pageable numpy cube, staged through the pinned ring)"}
    # The launch count runs last of all (main): the profiler's CUPTI session slows every later
    # host-side call of the process (the transform's numpy leg ran at a third of its rate behind it).
    def count(head):
        n_launch, names = count_launches(lambda: sp_w_svd_device(x, r, L, out=out))
        head["gpu_launches"] = n_launch * args.steps
        head["launch_names"] = names

    return {"ms": ms, "value": N * args.steps / (ms * 1e-3), "roofline": roofline, "e2e": e2e,
            "gpu_launches": None, "launch_names": None, "count_launches": count, "y_host": y_host,
            "k3_ms": k3_ms}


def headline_sharded(args, dist, sampler):
    """Strong scaling: one cube, rows sharded over the ranks (sharded.sp_w_svd_fused)."""
    import torch

    from paper_2601_08228_b200 import sharded as SH

    ws, rank = dist.get_world_size(), dist.get_rank()
    n1, n2, p = CFG4
    r, L = CFG4_RANK, CFG4_LEVELS
    N = n1 * n2 * p
    rows = SH.splits(n1, ws)
    r0 = sum(rows[:rank])
    if rank == 0:
        cube = torch.from_numpy(cfg4_cube()).cuda()
    else:
        cube = torch.empty(CFG4, dtype=torch.float64, device="cuda")
    dist.broadcast(cube, src=0)
    x = cube[r0:r0 + rows[rank]].contiguous()
    x_host = cube[r0:r0 + rows[rank]].cpu().pin_memory()
    del cube
    info = {}
    # The fused exchange (peer stores / loads through symmetric memory) has only ever run at world
    # size 1 on hardware (one GPU per round): check it once against the NCCL all-to-all variant and
    # fall back to that one -- on every rank together -- if it raises or disagrees, so a scaling run
    # still measures the sharded path.  The choice is reported in `exchange`.
    y_nccl = SH.sp_w_svd_sharded(x, r, L, n1)
    fused_ok, why = 1, None
    try:
        y_fused = SH.sp_w_svd_fused(x, r, L, n1)
        torch.cuda.synchronize()
        err = float((y_fused - y_nccl).abs().max() / y_nccl.abs().max().clamp_min(1e-300))
        if not err <= 1e-10:
            fused_ok, why = 0, f"fused vs NCCL result differs by {err:.2e}"
        del y_fused
    except Exception as e:  # noqa: BLE001 (any failure of the untested-at-scale path selects the fallback)
        fused_ok, why = 0, f"{type(e).__name__}: {e}"[:200]
    del y_nccl
    flag = torch.tensor([fused_ok], dtype=torch.int32, device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    use_fused = bool(flag.item())
    call = (lambda: SH.sp_w_svd_fused(x, r, L, n1)) if use_fused else (lambda: SH.sp_w_svd_sharded(x, r, L, n1))

    def step(record):
        info["y"] = call()

    ms = timed_region(step, args.steps, args.warmup, dist, sampler)
    # per-phase device times of one call (events inside the fused exchange)
    phases = SH.sp_w_svd_fused(x, r, L, n1, phase_times=True)[1] if use_fused else {}
    ms_nccl = timed_region(lambda rec: SH.sp_w_svd_sharded(x, r, L, n1), 3, 1, dist)
    peak, src = fp64_peak()
    m = p >> L
    ks = SH.splits(2 * m, ws)
    flops = ks[rank] * svd_flops(n1, n2)
    k4 = phases.get("k4_ms") or 0.0
    ach = flops / (k4 * 1e-3) / 1e12 if k4 > 0 else 0.0
    roofline = {"bound": "tensor", "kernel": f"K4 on this rank's {ks[rank]} coarse 1024^2 slices (rank {rank})",
                "achieved": round(ach, 3), "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4),
                "peak_source": src, "traffic": None, "flops_per_launch": flops}
    y_pin = torch.empty_like(x_host).pin_memory()

    def e2e_step(record):
        xd = x_host.to("cuda", non_blocking=True)
        y = SH.sp_w_svd_fused(xd, r, L, n1) if use_fused else SH.sp_w_svd_sharded(xd, r, L, n1)
        y_pin.copy_(y, non_blocking=True)

    e2e_steps = max(1, min(args.steps, 5))
    e2e_ms = timed_region(e2e_step, e2e_steps, 1, dist)
    e2e = {"value": round(N * e2e_steps / (e2e_ms * 1e-3), 1), "unit": UNIT,
           "h2d_bytes_per_step": 8 * N, "d2h_bytes_per_step": 8 * N,
           "api": "per rank: its pinned host rows H2D, sharded.sp_w_svd_fused, its rows of the result D2H"}
    return {"ms": ms, "value": N * args.steps / (ms * 1e-3), "roofline": roofline, "e2e": e2e,
            "phases_ms_rank": phases, "nccl_variant_ms_per_call": ms_nccl / 3,
            "exchange": "fused peer stores / loads (symmetric memory)" if use_fused
            else f"NCCL all_to_all_single (fused path not used: {why or 'another rank reported a failure'})",
            "gpu_launches": None}


# ----------------------------------------------------------- transform ----

def transform_key(args, dist, rank, ws, with_cpu):
    """BASELINE configs[1]: forward + inverse lifting at L = 1, 2, 4, 8 on a
    resident 512x512x256 cube per rank (weak: one cube per rank), HBM GB/s."""
    import torch

    from paper_2601_08228_b200 import engine as E
    import paper_2601_08228_b200 as W

    n1, n2, p = CFG2
    N = n1 * n2 * p
    x_host = np.random.default_rng(rank).standard_normal(CFG2)
    x = torch.from_numpy(x_host).cuda()
    bufs = {L: torch.empty((p, n1, n2), dtype=torch.float64, device="cuda") for L in CFG2_LEVELS}
    y = torch.empty_like(x)
    ev = {"f": [], "i": []}

    def step(record):
        for L in CFG2_LEVELS:
            if record:
                for k, fn in (("f", lambda: E.lift_forward(x, L, out=bufs[L])),
                              ("i", lambda: E.lift_inverse(bufs[L], n1, n2, p, L, out=y))):
                    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    s.record()
                    fn()
                    e.record()
                    ev[k].append((s, e))
            else:
                E.lift_forward(x, L, out=bufs[L])
                E.lift_inverse(bufs[L], n1, n2, p, L, out=y)

    steps = max(3, min(args.steps, 10))
    ms = timed_region(step, steps, 2, dist)
    assert float((y - x).norm() / x.norm()) < 1e-12
    bytes_step = len(CFG2_LEVELS) * 2 * 16 * N
    peak, src = hbm_peak()
    f_ms = sum(s.elapsed_time(e) for s, e in ev["f"]) / len(ev["f"])
    i_ms = sum(s.elapsed_time(e) for s, e in ev["i"]) / len(ev["i"])
    per = 16 * N
    af, ai = per / (f_ms * 1e-3) / 1e9, per / (i_ms * 1e-3) / 1e9
    out = {"config": "forward+inverse lifting 512x512x256 f64, L=1,2,4,8 per step (BASELINE configs[1]); "
                     "one cube per rank", "metric": "HBM GB/s (algorithmic 16 B per element per direction)",
           "value": round(ws * bytes_step * steps / (ms * 1e-3) / 1e9, 2), "unit": "GB/s", "steps": steps,
           "roofline": {"bound": "hbm", "kernel": "K2_inverse" if i_ms >= f_ms else "K1_forward",
                        "achieved": round(min(af, ai), 1), "peak": peak, "unit": "GB/s",
                        "frac": round(min(af, ai) / peak, 4), "peak_source": src,
                        "traffic": profile_value("K2_inverse" if i_ms >= f_ms else "K1_forward",
                                                 "dram_bytes_per_launch"),
                        "algorithmic_bytes_per_launch": per,
                        "per_kernel": {"K1_forward": {"ms": round(f_ms, 4), "GBps": round(af, 1),
                                                      "frac": round(af / peak, 4)},
                                       "K2_inverse": {"ms": round(i_ms, 4), "GBps": round(ai, 1),
                                                      "frac": round(ai / peak, 4)}}}}
    # public API on host arrays (pyramid returned to the host, then inverted from it);
    # two warm-up passes fill the caching host allocator's pinned blocks
    x_pin = W.pinned_empty(x_host.shape)  # the cube in page-locked memory: uploaded by DMA in place
    x_pin[...] = x_host
    for _ in range(2):  # (as the timed loop: the previous result alive while the next call runs, so
        for L in CFG2_LEVELS:  # the pool's third pinned result buffer is page-locked here, not there)
            o = W.inverse_w(W.forward_w(x_pin, L))
    dts = []
    for _ in range(3):  # median of three passes (a pass that page-locks a new pooled buffer costs +0.2 s)
        t = time.perf_counter()
        for L in CFG2_LEVELS:
            o = W.inverse_w(W.forward_w(x_pin, L))
        dts.append(time.perf_counter() - t)
    dt = sorted(dts)[1]
    assert float(np.linalg.norm((o - x_host).ravel()) / np.linalg.norm(x_host.ravel())) < 1e-12
    out["e2e"] = {"value": round(bytes_step / dt / 1e9, 2), "unit": "GB/s",
                  "api": "inverse_w(forward_w(numpy cube in page-locked memory, L)) for L = 1, 2, 4, 8 "
                         "(pyramid returned to host); median of 3 passes",
                  "h2d_bytes_per_step": len(CFG2_LEVELS) * 16 * N, "d2h_bytes_per_step": len(CFG2_LEVELS) * 16 * N}
    if with_cpu:
        from oracle import parallel as P

        def run(pool):
            for L in CFG2_LEVELS:
                s, d = P.lift_forward(pool, x_host, L)
                P.lift_inverse(pool, s, d)

        out["cpu_baseline"] = cpu_port_baseline(run, lambda s: round(bytes_step / s / 1e9, 3), "GB/s",
                                                "oracle forward + inverse transform, L = 1, 2, 4, 8, rows split "
                                                "over the threads", reps=2)
    return out


# ----------------------------------------------------------- workloads ----

def wsvd_workload(args, steps=5, warmup=3):
    """Config 3: w_svd rank 20 of the 256x256x192 cube, L = 3."""
    import torch

    from paper_2601_08228_b200 import engine as E
    from paper_2601_08228_b200 import synth
    from paper_2601_08228_b200.decomposition import w_svd_device
    import paper_2601_08228_b200 as W

    n1, n2, p, r, L = 256, 256, 192, 20, 3
    x_host = synth.hyperspectral_cube(n1, n2, p, seed=0)
    x = torch.from_numpy(x_host).cuda()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    info = {}
    with PhaseTimer() as pt:
        def step(record):
            flush.zero_()  # 256 MB > L2: every call starts cold
            pt.on = record
            info["out"] = w_svd_device(x, r, L)
            pt.on = False
            info["sweeps"] = E.last_sweeps()

        ms = timed_region(step, steps, warmup)
        k4 = pt.total_ms("svd") / max(pt.calls("svd"), 1)
    call_ms = ms / steps
    N = n1 * n2 * p
    flops = p * svd_flops(n1, n2)
    peak, src = fp64_peak()
    ach = flops / (k4 * 1e-3) / 1e12
    recon = info["out"][4].cpu().numpy()
    from oracle import parallel as P

    ref = {}

    def run(pool):
        ref["o"] = P.w_svd(pool, x_host, r, L)

    cpu = cpu_port_baseline(run, lambda s: round(N / s, 1), UNIT, "oracle w_svd(cube, 20, 3)")
    rel = float(np.linalg.norm((recon - ref["o"]["recon"]).ravel()) / np.linalg.norm(ref["o"]["recon"].ravel()))
    return {"config": "w_svd 256x256x192 rank 20 L=3 (BASELINE configs[2])", "metric": UNIT,
            "value": N / (call_ms * 1e-3), "ms_per_call": call_ms, "jacobi_sweeps": info["sweeps"],
            "roofline": {"bound": "tensor", "kernel": "K4 (192 wavelet slices 256^2)", "achieved": round(ach, 3),
                         "peak": peak, "unit": "TFLOP/s", "frac": round(ach / peak, 4), "peak_source": src,
                         "k4_ms_per_call": round(k4, 3),
                         "flops_model": "192 x (14 m n^2 + 8 n^3) Golub-Kahan thin-SVD count (SURVEY 8d)"},
            "l2": "256 MB flush before each call",
            "e2e": {"ms_per_call": round(api_e2e(lambda: W.w_svd(x_host, r, L), 2), 2),
                    "api": "w_svd(numpy cube, 20, 3) -> (SvdFactors of numpy arrays, numpy recon)",
                    "h2d_bytes_per_call": 8 * N, "d2h_bytes_per_call": 8 * (N + p * (n1 + n2 + r) * r)},
            "cpu_baseline": cpu, "recon_relerr_vs_cpu": rel}


def api_e2e(fn, reps):
    """Wall ms of a synchronous public-API call on host (numpy) inputs (H2D and D2H inside)."""
    import torch

    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps * 1e3


def deblur_workload(args, steps=3, warmup=3):
    """Config 5: w-pinv deblurring recovery (2 pinv_w + 2 w_product), 512x512x128, L = 3."""
    import torch

    import paper_2601_08228_b200 as W
    from paper_2601_08228_b200 import imaging, synth
    from paper_2601_08228_b200.algebra import w_product_device
    from paper_2601_08228_b200.decomposition import pinv_w_device_many

    x, av, ah, eta = synth.deblur_problem()
    xd, avd, ahd = (torch.from_numpy(t).cuda() for t in (x, av, ah))
    aht = W.transpose(ahd)
    b = w_product_device(w_product_device(avd, xd, 3), aht, 3) + torch.from_numpy(eta).cuda()
    res = {}
    with PhaseTimer() as pt:
        def step(record):
            pt.on = record
            # imaging.deblur's device path: both pseudo-inverses in one batched K4 call
            left, right = pinv_w_device_many([avd, aht], 3, 1e-3)
            res["x"] = w_product_device(w_product_device(left, b, 3), right, 3)
            pt.on = False

        ms = timed_region(step, steps, warmup)
        k4 = pt.total_ms("svd") / max(pt.calls("svd"), 1)
    # the face GEMM of one w-product (K3 over the 128 wavelet slices of 512^2), timed alone
    from paper_2601_08228_b200 import engine as E

    pa = E.lift_forward(xd.contiguous(), 3)
    pb = E.lift_forward(avd.contiguous(), 3)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    E.gemm(pa, pb)
    ev[0].record()
    for _ in range(5):
        E.gemm(pa, pb)
    ev[1].record()
    torch.cuda.synchronize()
    k3 = ev[0].elapsed_time(ev[1]) / 5
    peak, src = fp64_peak()
    svd_f = 2 * 128 * svd_flops(512, 512)
    nz_f = 2 * 16 * svd_flops(512, 512)  # slice-constant operators: 16 nonzero (smooth) wavelet slices each
    gemm_f = 2 * 512 ** 3 * 128
    xr = res["x"].cpu().numpy()
    b_host = b.cpu().numpy()
    from oracle import parallel as P
    from oracle import wten_oracle as O

    ref = {}

    def run(pool):
        ref["x"] = P.deblur(pool, b_host, av, O.transpose(ah), 3, 1e-3)

    cpu = cpu_port_baseline(run, lambda s: round(s, 3), "s per recovery",
                            "oracle recovery w_product(w_product(pinv_w(A_V), B), pinv_w(A_H^T)), L=3, tol 1e-3")
    rel = float(np.linalg.norm((xr - ref["x"]).ravel()) / np.linalg.norm(ref["x"].ravel()))
    return {"config": "w-pinv deblur 512x512x128, 9x9 Gaussian PSF sigma=2, L=3, tol 1e-3 (BASELINE configs[4])",
            "metric": "s per recovery", "value": ms / steps / 1e3, "higher_is_better": False,
            "psnr_db": imaging.psnr(xd, res["x"]), "ssim": imaging.ssim(xd, res["x"]),
            "psnr_db_blurred_input": imaging.psnr(xd, b), "ssim_blurred_input": imaging.ssim(xd, b),
            "quality_note": ("PSNR paper-verbatim 10 log10(N MPP / ||e||^2) (PAPER.md:878). Under the lazy-wavelet "
                             "w-product a slice-constant operator has zero detail blocks, so blur keeps only the "
                             "8-band means and the 9x9 sigma=2 Toeplitz operators amplify the noise up to 1e3x "
                             "per side: the recovery is poor by construction of the config"),
            "roofline_k4_pinv": {"bound": "tensor", "kernel": "K4 on both operators' 256 wavelet slices of 512^2 "
                                 "(224 exactly zero: retired before any work)",
                                 "achieved": round(nz_f / (k4 * 1e-3) / 1e12, 3), "peak": peak, "unit": "TFLOP/s",
                                 "frac": round(nz_f / (k4 * 1e-3) / 1e12 / peak, 4), "peak_source": src,
                                 "k4_ms_per_call": round(k4, 3),
                                 "flops_model": "32 nonzero slices x (14 m n^2 + 8 n^3), m = n = 512",
                                 "effective_frac_dense": round(svd_f / (k4 * 1e-3) / 1e12 / peak, 4),
                                 "effective_note": "on the dense count the reference executes (2 x 128 slices, the "
                                                   "zero ones included)"},
            "roofline_k3_face_gemm": {"bound": "tensor", "kernel": "K3 face GEMM (128 x 512^3 per w-product)",
                                      "achieved": round(gemm_f / (k3 * 1e-3) / 1e12, 3) if k3 else None,
                                      "peak": peak, "unit": "TFLOP/s",
                                      "frac": round(gemm_f / (k3 * 1e-3) / 1e12 / peak, 4) if k3 else None,
                                      "k3_ms_per_call": round(k3, 4),
                                      "note": "K3 over the 128 wavelet slices of one w-product (512^3 each), timed "
                                              "alone with CUDA events, 5 calls"},
            "cpu_baseline": cpu, "recovery_relerr_vs_cpu": rel}


def wproduct_workload(args, steps=50, warmup=5):
    """Config 1: w_product 64x48x32 * 48x40x32, L = 1 (latency-bound)."""
    import torch

    from paper_2601_08228_b200 import synth
    from paper_2601_08228_b200.algebra import w_product_device
    import paper_2601_08228_b200 as W

    a, b = synth.uniform_pair(0)
    ad, bd = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()

    def step(record):
        w_product_device(ad, bd, 1)

    ms = timed_region(step, steps, warmup)
    from oracle import wten_oracle as O

    cpu_s, ts = cpu_median(lambda: O.w_product(a, b, 1), reps=5, warm=2)
    return {"config": "w_product 64x48x32 * 48x40x32 L=1 (BASELINE configs[0])", "metric": "us per call",
            "value": ms / steps * 1e3, "higher_is_better": False,
            "roofline": {"bound": "latency", "note": "7.9 MFLOP and 3.9 MB per call: four launches "
                         "(K1, K1, K3, K2) and their host overhead set the time"},
            "e2e_us": round(api_e2e(lambda: W.w_product(a, b, 1), 20) * 1e3, 1),
            "cpu_baseline": {"value": round(cpu_s * 1e6, 1), "unit": "us per call", "cores": 1, "kind": "port",
                             "sample": "oracle w_product (numpy, one thread: the call is too small to split), "
                                       "2 warm-ups + median of 5, full size"}}


def comparators_workload(args):
    """Paper-style ratios on B200: w- vs t- vs m-product on a
    p = 256 cube and w-svd / sp-w-svd vs t-svd on the config-3 cube, device-resident."""
    import torch

    import paper_2601_08228_b200 as W
    from paper_2601_08228_b200 import baselines as B, synth

    p = 256
    g = torch.Generator(device="cuda").manual_seed(7)
    a = torch.randn((p, p, p), dtype=torch.float64, device="cuda", generator=g)
    b = torch.randn((p, p, p), dtype=torch.float64, device="cuda", generator=g)
    tr = B.dct_transform(p)
    L = W.max_levels(p)
    out = {"config": f"cube {p}^3 products (L={L}); w_svd / sp_w_svd / t_svd on 256x256x192 r=20 L=3",
           "metric": "ms per call (device-resident)"}
    for k, fn in (("w_product", lambda: W.w_product(a, b, L)), ("t_product", lambda: B.t_product(a, b)),
                  ("m_product", lambda: B.m_product(a, b, tr))):
        out[k + "_ms"] = timed_region(lambda rec: fn(), 5, 2) / 5
    x = torch.from_numpy(synth.hyperspectral_cube(256, 256, 192, seed=0)).cuda()
    for k, fn in (("w_svd", lambda: W.w_svd(x, 20, 3)), ("sp_w_svd", lambda: W.sp_w_svd(x, 20, 3)),
                  ("t_svd", lambda: B.t_svd(x, 20))):
        out[k + "_ms"] = timed_region(lambda rec: fn(), 3, 1) / 3
    out["speedup_w_vs_t_product"] = out["t_product_ms"] / out["w_product_ms"]
    out["speedup_w_vs_t_svd"] = out["t_svd_ms"] / out["w_svd_ms"]
    out["speedup_spw_vs_t_svd"] = out["t_svd_ms"] / out["sp_w_svd_ms"]
    out["op_counts"] = {k: B.op_count(k, p, p, p, p).count for k in "mtw"}
    return out


# ------------------------------------------------------- reference arm ----

def run_reference(args):
    """The reference algorithm (oracle port: numpy + LAPACK dgesdd over all host
    threads, oracle/parallel.py) on the headline workload; rank 0 only."""
    ws, rank, local = dist_env()
    if rank != 0:
        return
    from oracle import parallel as P

    x = cfg4_cube()
    n1, n2, p = CFG4
    N = n1 * n2 * p
    with P.Pool() as pool:
        def call():
            P.sp_w_svd(pool, x, CFG4_RANK, CFG4_LEVELS)

        t = time.perf_counter()
        call()  # first warm-up call sizes the run
        first = time.perf_counter() - t
        budget = float(os.environ.get("WT_REF_BUDGET_S", "420"))
        warm, steps, note = args.warmup, args.steps, None
        if first * (warm - 1 + steps) > budget:
            # bounded run on a slow host: no further warm-ups, as many full calls as fit
            warm = 1
            steps = max(1, min(steps, int(budget / first)))
            note = (f"time budget {budget:.0f} s at {first:.1f} s per call: {steps} of {args.steps} steps "
                    f"timed after 1 warm-up")
        for _ in range(warm - 1):
            call()
        t = time.perf_counter()
        for _ in range(steps):
            call()
        dt = time.perf_counter() - t
        threads = pool.threads
    v = N * steps / dt
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 1), "unit": UNIT, "n_gpus": args.gpus,
            "steps": steps, "warmup": args.warmup, "ms_per_step": round(dt / steps * 1e3, 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": headline_config(),
            "cpu_baseline": {"value": round(v, 1), "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": "oracle/parallel.py sp_w_svd (numpy port of decomposition.py:140-154, "
                                       f"LAPACK dgesdd per slice) on the full cube over {threads} host threads, "
                                       "one full call per step"},
            "e2e": {"value": round(v, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if note:
        line["note"] = note
    emit(line)


# ----------------------------------------------------------------- main ----

_JSON_FD = None


def _quiet_stdout():
    """Send everything written to fd 1 (NCCL's banner, library prints) to stderr;
    the JSON line goes to the saved stdout so it stays the only line."""
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    _quiet_stdout()
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    ws, rank, local = dist_env()
    import torch

    torch.cuda.set_device(local)
    dist = None
    if ws > 1 or args.force_dist:
        import torch.distributed as tdist

        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist
    from paper_2601_08228_b200 import _native

    _native.require_gpu()
    n1, n2, p = CFG4
    N = n1 * n2 * p
    sampler = ClockSampler(torch.cuda.current_device())
    if dist is None:
        x_host = cfg4_cube()
        head = headline_single(args, x_host, sampler)
    else:
        x_host = None
        head = headline_sharded(args, dist, sampler)

    if args.workloads == "default":
        wl = ["wsvd", "deblur", "wproduct", "comparators"] if dist is None else []
    elif args.workloads == "none":
        wl = []
    else:
        wl = [w for w in args.workloads.split(",") if w]
    want_cpu = rank == 0 and dist is None and not args.no_cpu_baseline

    cpu = None
    if want_cpu:
        ref = {}

        def run(pool):
            from oracle import parallel as P

            ref["y"] = P.sp_w_svd(pool, x_host, CFG4_RANK, CFG4_LEVELS)

        cpu = cpu_port_baseline(run, lambda s: round(N / s, 1), UNIT,
                                "oracle sp_w_svd(cube, 30, 4) (decomposition.py:140-154)")
        y = head["y_host"]
        cpu["gpu_vs_cpu_recon_relerr"] = float(np.linalg.norm((y - ref["y"]).ravel())
                                               / np.linalg.norm(ref["y"].ravel()))
        del ref

    transform = transform_key(args, dist, rank, ws, want_cpu)
    workloads = {}
    budget = float(os.environ.get("WT_BENCH_WORKLOAD_TIMEOUT", "900"))
    t_start = time.time()
    for name in wl:
        if time.time() - t_start > budget:
            workloads[name] = {"skipped": f"workload budget {budget:.0f} s spent"}
            continue
        try:
            fn = {"wsvd": wsvd_workload, "deblur": deblur_workload, "wproduct": wproduct_workload,
                  "comparators": comparators_workload}[name]
            workloads[name] = fn(args)
        except Exception as e:  # noqa: BLE001
            workloads[name] = {"error": f"{type(e).__name__}: {e}"}

    if head.get("count_launches"):
        head["count_launches"](head)
    if rank == 0:
        line = {
            "metric": METRIC, "value": round(head["value"], 1), "unit": UNIT, "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(head["ms"] / args.steps, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": DATA,
            "config": headline_config(),
            "parallelism": "single GPU" if dist is None else f"rows sharded over {ws} GPUs ({head.get('exchange', 'fused')})",
            "roofline": head["roofline"],
            "cpu_baseline": cpu,
            "e2e": head["e2e"],
            "gpu_launches": head["gpu_launches"],
            "clocks": sampler.summary(),
            "transform": transform,
            "workloads": workloads,
        }
        for k in ("phases_ms_rank", "nccl_variant_ms_per_call", "exchange", "launch_names"):
            if k in head:
                line[k] = head[k]
        emit(line)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
