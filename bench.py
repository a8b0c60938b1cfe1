#!/usr/bin/env python
"""OSBF benchmark (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload C1..C5] [--mode fast|exact] [--radius R]

A *step* is one full run of the hot path over one workload: ``iterations``
Jacobi OSBF passes (osbf::osbf, filters2d.hpp:91-98) with the input resident
in HBM.

Default workload: BASELINE config C5 — one 32768 x 32768 float32 image
(4 GiB), r = 4, 50 iterations — the largest configuration that fits one GPU
(BASELINE.json quotes its metric over 1/2/4/8 GPUs without naming a config).
At N = 1 the whole image runs through the C ABI (osbf_gpu_iterate); at N > 1
it is split into row bands, one per GPU, with the r-row halo exchanged every
pass (fused into the pass kernel through symmetric memory, NCCL send/recv as
the fallback): strong scaling over the same image.  ``--workload C4`` runs
the batch-sharded 256 x 1024^2 config (weak scaling).

Rank 0 prints ONE JSON line.  Timing: CUDA events on the launching stream,
max over ranks; every buffer (8.6 GB per fp64 plane) is larger than L2 (C4:
L2 flushed between steps); nvidia-smi clocks sampled during the timed region.
``e2e`` = the same metric through the C ABI host entry point the drop-in
headers call (osbf_gpu_osbf_host) from pinned host buffers, H2D + D2H inside
the timing.  At N = 1 the line carries sub-records, each with its own clocks:
``C4`` (256 x 1024^2, r=2, 20 it), ``r_sweep`` (one pass of the 32768^2
plane per r, the north star's flatness check) and ``C3`` (4096^2 uint8,
10 it, per r).  ``--impl reference`` times the reference's own CPU
implementation (the unmodified reference headers compiled into oracle/_ref).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "OSBF megapixel-iterations/sec and achieved HBM GB/s vs peak, 1/2/4/8 B200"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
           0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
           0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
           0x100: "display_clock_setting"}
IN_BYTES = {"u8": 1, "f32": 4, "f64": 8}
SWEEP_RADII = (1, 2, 4, 8, 16)
C5_SWEEP_RADII = (1, 2, 3, 4, 6, 8, 12, 16, 24, 32)  # > 16: the exact table path (whole planes)


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="C5", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--mode", choices=["fast", "exact"], default="fast")
    ap.add_argument("--radius", type=int, default=None)
    ap.add_argument("--iterations", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the C4 / sweep sub-records")
    ap.add_argument("--c5-scaling", choices=("strong", "weak"), default="strong",
                    help="C5 over N GPUs: the fixed 32768^2 image (strong) or a 32768 x 4096 "
                         "band per GPU, 32768 x 4096N in total (weak, SURVEY §8e)")
    ap.add_argument("--exchange", choices=("push", "nccl"), default="push",
                    help="C5 halo exchange: fused into the pass kernel (symmetric memory) "
                         "or NCCL send/recv after it")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args(argv)


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce(x: float, world: int, op: str = "max") -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = os.path.join("/tmp", f"osbf_clocks_{os.getpid()}_{id(self)}.csv")

    def start(self):
        try:
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,power.draw",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        sm, smax, reasons, power = [], [], set(), []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 4:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
                mask = int(parts[2], 16) if parts[2].startswith("0x") else int(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for bit, name in REASONS.items():
                if mask & bit and name != "gpu_idle":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


def hbm_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM_GBS, "fallback"


def ncu_traffic(workload: str, mode: str, kernel: str):
    """Per-launch DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of
    the dominant kernel from the committed ncu --set full summary
    (profiles/ncu_summary.json, keyed workload/mode/kernel), if one exists."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d[f"{workload}/{mode}/{kernel}"]["dram_bytes_per_launch"]
    except (OSError, KeyError, ValueError):
        return None


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_desc(cfg, r, iters):
    return (f"{cfg.name}: {cfg.batch} x {cfg.height}x{cfg.width} {cfg.dtype} seeded synthetic "
            f"mosaic+noise, r={r}, {iters} iterations")


def roofline(alg_bytes_per_launch: float, launch_ms: float, kernel: str, workload: str,
             mode: str, rule: str):
    peak, peak_kind = hbm_peak()
    achieved = alg_bytes_per_launch / (launch_ms / 1000.0) / 1e9
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "peak_kind": peak_kind,
            "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": ncu_traffic(workload, mode, kernel), "kernel": kernel,
            "algorithmic_bytes_per_launch": int(alg_bytes_per_launch),
            "avg_launch_ms": round(launch_ms, 5), "bytes_rule": rule}


def time_steps(run, steps, stream, pre=None):
    """CUDA-event time of ``steps`` calls of run() on ``stream`` (ms each)."""
    import torch

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        if pre is not None:
            pre(i)
        starts[i].record(stream)
        run()
        ends[i].record(stream)
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in zip(starts, ends)]


# ---- CPU reference (oracle/_ref: the unmodified reference headers) ---------

def reference_runner(threads: int):
    import oracle

    if oracle.Reference.available():
        ref = oracle.Reference()
        ref.pin_allocator_for_timing()
        ref.set_max_threads(threads)
        return (lambda p, r, it: ref.osbf(p, r, it)), "reference"  # noqa: E731
    orc = oracle.Oracle()
    return (lambda p, r, it: orc.osbf(p, r, it, threads=threads)), "port"  # noqa: E731


def cpu_rate(plane, r, threads, reps=3):
    """Median Mpx-iter/s of the reference's osbf(plane, r, 1) on ``threads``
    host threads, after a >= 1 s warm-up."""
    import numpy as np

    run, kind = reference_runner(threads)
    p = np.ascontiguousarray(plane, dtype=np.float64)
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        run(p[:256, :256], r, 1)
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        run(p, r, 1)
        ts.append(time.perf_counter() - t0)
    return p.size / statistics.median(ts) / 1e6, kind, statistics.median(ts)


def cpu_baseline_c5(x_host, r):
    threads = os.cpu_count() or 1
    v, kind, t = cpu_rate(x_host[:4096], r, threads)
    v1, _, t1 = cpu_rate(x_host[:512], r, 1)
    return {"value": round(v, 3), "unit": "Mpx-iter/s", "cores": threads, "kind": kind,
            "sample": f"reference osbf::osbf, 1 pass over a 4096x32768 slice of C5 (r={r}), "
                      f"median of 3 ({t:.2f} s each), {threads} threads; per-iteration cost "
                      "is constant, so the rate holds for 50 iterations",
            "one_thread": {"value": round(v1, 3), "unit": "Mpx-iter/s", "cores": 1,
                           "sample": f"1 pass over a 512x32768 slice, median of 3 ({t1:.2f} s)"},
            "cpu_model": cpu_model()}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU path, rank 0 only; each step a
    bounded sample of the workload (per-iteration cost is constant)."""
    if rank != 0:
        return
    import numpy as np

    from paper_2108_05021_b200 import synth

    cfg = synth.CONFIGS[args.workload]
    r = args.radius or cfg.radius
    iters = args.iterations or cfg.iterations
    threads = os.cpu_count() or 1
    run, kind = reference_runner(threads)
    if args.workload == "C5":
        rng = np.random.default_rng(5)
        n = max(8, int(3 * 2048 * 32768 / (264.0 * 264.0)))
        sample = synth.add_noise_f32(synth.rect_mosaic(2048, 32768, rng, n_rects=n,
                                                       size=(16, 512)), 0.05, rng)
        planes = [sample]
        desc = "per step: 1 pass over a 2048x32768 C5-style slice"
        it_per_step = 1
    else:
        x = synth.make_input(args.workload)
        planes = list(x.reshape(-1, x.shape[-2], x.shape[-1]))
        desc = None
        it_per_step = None
    p0 = np.asarray(planes[0], dtype=np.float64)
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        run(p0[:256, :256], r, 1)
    if it_per_step is None:
        t0 = time.perf_counter()
        run(p0, r, 1)
        t_it = time.perf_counter() - t0
        it_per_step = int(max(1, min(iters, 1.5 / max(t_it, 1e-6))))
        desc = (f"per step: 1 plane of {p0.shape[0]}x{p0.shape[1]} x {it_per_step} of {iters} "
                "iterations")
    px_step = p0.size * it_per_step
    for i in range(args.warmup):
        run(np.asarray(planes[i % len(planes)], dtype=np.float64), r, it_per_step)
    times = []
    for i in range(args.steps):
        p = np.asarray(planes[i % len(planes)], dtype=np.float64)
        t0 = time.perf_counter()
        run(p, r, it_per_step)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    value = px_step * args.steps / total / 1e6
    sample = f"{desc} (per-iteration cost is constant), {threads} threads, {cpu_model()}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "Mpx-iter/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * total / args.steps, 3), "higher_is_better": True,
        "scaling": "strong" if args.workload == "C5" else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, r, iters), "radius": r, "iterations": iters,
                   "parallelism": "cpu threads"},
        "cpu_baseline": {"value": round(value, 3), "unit": "Mpx-iter/s", "cores": threads,
                         "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "Mpx-iter/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }), flush=True)


# ---- sub-records (N = 1) ----------------------------------------------------

def sub_c4(ctx, steps):
    import torch

    from paper_2108_05021_b200 import synth

    x = torch.from_numpy(synth.make_input("C4")).cuda()
    y = torch.empty(x.shape, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ctx.iterate(x, 2, 20, mode="fast", out=y)
    clk = ClockSampler(torch.cuda.current_device()).start()
    ms = time_steps(lambda: ctx.iterate(x, 2, 20, mode="fast", out=y), steps,
                    torch.cuda.current_stream(), pre=lambda i: flush.fill_(i & 0xFF))
    c = clk.stop()
    step = sum(ms) / len(ms)
    px = x.numel()
    rl = roofline(px * ((4 + 8) + 19 * 16) / 20, step / 20, ctx.last_kernel, "C4", "fast",
                  "read U^t + write U^{t+1}: first pass 4+8 B, then 8+8 B")
    return {"workload": "C4: 256 x 1024^2 f32, r=2, 20 iterations, fast, L2 flushed between steps",
            "value": round(px * 20 / (step / 1000) / 1e6, 3), "unit": "Mpx-iter/s",
            "ms_per_step": round(step, 4), "roofline": rl, "clocks": c}


def sub_sweep(ctx, x, workload, iters, radii, in_bytes, reps=5, mode="fast"):
    """One record per radius, each with its own clocks: ``iters`` passes in
    ``mode`` over ``x`` (fp64 storage between passes)."""
    import torch

    y = torch.empty(x.shape, dtype=torch.float64, device="cuda")
    out = []
    px = x.numel()
    for r in radii:
        for _ in range(2):
            ctx.iterate(x, r, iters, mode=mode, out=y)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.iterate(x, r, iters, mode=mode, out=y)
        torch.cuda.synchronize()
        n = max(reps, int(0.8 / max(time.perf_counter() - t0, 1e-4)))  # >= ~0.8 s sampled
        clk = ClockSampler(torch.cuda.current_device()).start()
        ms = time_steps(lambda: ctx.iterate(x, r, iters, mode=mode, out=y), n,
                        torch.cuda.current_stream())
        c = clk.stop()
        step = statistics.median(ms)
        alg = px * ((in_bytes + 8) + (iters - 1) * 16) / iters
        out.append({"r": r, "value": round(px * iters / (step / 1000) / 1e6, 3),
                    "unit": "Mpx-iter/s", "ms_per_pass": round(step / iters, 5),
                    "kernel": ctx.last_kernel,
                    "frac": round(alg / (step / iters / 1000) / 1e9 / hbm_peak()[0], 4),
                    "clocks": {"sm_mhz": c.get("sm_mhz"), "reasons": c.get("reasons")}})
    return {"workload": workload, "records": out}


# ---- C5 (the default) -----------------------------------------------------------

def run_c5(args, world, rank, local):
    import ctypes

    import torch

    import paper_2108_05021_b200 as ob
    from paper_2108_05021_b200 import synth
    from paper_2108_05021_b200.dist import BandLayout, RowBandOSBF

    torch.cuda.set_device(local)
    cfg = synth.CONFIGS["C5"]
    r = args.radius or cfg.radius
    iters = args.iterations or cfg.iterations
    mode = args.mode
    W = 32768
    H = 4096 * world if args.c5_scaling == "weak" else 32768
    x = synth.make_c5_on_device(H, W, seed=5)  # identical on every rank (Philox)
    stream = torch.cuda.current_stream()
    ctx = ob.Context(local)
    runner = None
    if world == 1:
        y = torch.empty((H, W), dtype=torch.float64, device="cuda")

        def step():
            ctx.iterate(x, r, iters, mode=mode, out=y)
        rows = H
    else:
        if mode != "fast":
            raise SystemExit("row bands partition the fast mode only (SURVEY §8e)")
        lay = BandLayout.make(H, W, r, world, rank)
        band = x[lay.row0:lay.row1]
        runner = RowBandOSBF(lay, rank, world, exchange=args.exchange)

        def step():
            runner.run(band, iters)
        rows = lay.rows
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    kctx = runner._ctx if runner is not None else ctx
    kernel = kctx.last_kernel
    launches0 = kctx.launches
    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ms = time_steps(step, args.steps, stream)
    barrier(world)
    clk = clocks.stop()
    launches = int(allreduce(kctx.launches - launches0, world, "sum"))
    total_ms = allreduce(sum(ms), world, "max")
    value = H * W * iters * args.steps / (total_ms / 1000.0) / 1e6
    pass_ms = sum(ms) / (args.steps * iters)  # this rank's average launch (incl. exchange)
    in_b = 4 if world == 1 else 8  # bands start from a fp64 copy of the rank's rows
    alg = rows * W * ((in_b + 8) + (iters - 1) * 16) / iters
    exch = (runner.exchange if runner is not None else "none (1 rank)")
    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpx-iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": args.c5_scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, r, iters) + (
                       f" (weak: {W} x {H} = 4096 rows per GPU)" if args.c5_scaling == "weak"
                       else ""), "height": H, "width": W, "radius": r, "iterations": iters,
                   "mode": mode, "storage": "f64 between passes (float32 input read on the "
                                            "first pass)",
                   "parallelism": "whole image, one GPU" if world == 1 else
                   f"row bands x{world}, {r}-row halo exchange per pass ("
                   + ("fused into the pass kernel: stores into the neighbours' "
                      "symmetric-memory halos + device barrier" if exch == "push"
                      else "NCCL send/recv") + ")",
                   "l2": "every buffer (8.6 GB fp64 plane) larger than the 126 MB L2"},
        "roofline": roofline(alg, pass_ms, kernel, "C5", mode,
                             "read U^t + write U^{t+1} per pass: first pass 4+8 B (float32 "
                             "input), then 8+8 B; avg launch = step time / iterations"),
        "gpu_launches": launches,
        "launches_per_pass": round(launches / max(1, args.steps * iters * world), 3),
        "clocks": clk,
        "exchange": exch,
    }
    if runner is not None and runner.exchange_note:
        result["exchange_note"] = runner.exchange_note

    x_host = None
    if not args.no_e2e:
        # end to end through the C ABI host entry point (what the drop-in
        # osbf::osbf calls): pinned float32 input -> H2D -> passes -> D2H of
        # the fp64 result, every step
        if world == 1:
            x_host = x.cpu().pin_memory()
            h_out = torch.empty((H, W), dtype=torch.float64).pin_memory()
            lib = ctx._lib
            mcode = {"exact": 0, "fast": 1}[mode]

            def e2e_call():
                st = lib.osbf_gpu_osbf_host(ctx.handle, 1, ctypes.c_void_p(x_host.data_ptr()),
                                            ctypes.c_void_p(h_out.data_ptr()), W, H, 1, r, iters,
                                            mcode)
                if st != 0:
                    raise RuntimeError(lib.osbf_gpu_last_error().decode())
            h2d, d2h = x_host.numel() * 4, H * W * 8
            api = "osbf_gpu_osbf_host (C ABI, pinned host buffers)"
        else:
            b_host = band.cpu().pin_memory()
            h_out = torch.empty((lay.rows, W), dtype=torch.float64).pin_memory()
            d_band = torch.empty_like(band)

            def e2e_call():
                d_band.copy_(b_host, non_blocking=True)
                res = runner.run(d_band, iters)
                h_out.copy_(res, non_blocking=True)
                torch.cuda.synchronize()
            h2d, d2h = b_host.numel() * 4, lay.rows * W * 8
            api = "row-band runner from pinned host rows (H2D band, passes, D2H band)"
        e2e_call()
        e2e_steps = max(1, min(args.steps, 3))
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_call()
        torch.cuda.synchronize()
        dt = allreduce(time.perf_counter() - t0, world, "max")
        result["e2e"] = {"value": round(H * W * iters * e2e_steps / dt / 1e6, 3),
                         "unit": "Mpx-iter/s", "h2d_bytes_per_step": int(h2d * world),
                         "d2h_bytes_per_step": int(d2h * world), "steps": e2e_steps, "api": api}
        if world == 1:
            result["e2e"]["matches_device_path"] = bool(
                torch.equal(h_out.view(torch.int64), y.cpu().view(torch.int64)))
    else:
        result["e2e"] = None

    if world == 1 and rank == 0 and not args.no_sub:
        del y
        torch.cuda.empty_cache()
        subs = {"C4": sub_c4(ctx, max(3, min(args.steps, 10)))}
        xf = x.double()
        subs["r_sweep"] = sub_sweep(ctx, xf, "one fast pass of the 32768^2 C5 plane (fp64 in "
                                    "and out) per radius: the r-flatness check",
                                    1, C5_SWEEP_RADII, 8)
        del xf
        torch.cuda.empty_cache()
        c3 = torch.from_numpy(synth.make_input("C3")[0]).cuda()
        subs["C3"] = sub_sweep(ctx, c3, "C3: 4096^2 uint8, 10 fast iterations per radius "
                               "(first pass bit-exact; plane fits L2: per-pass figure is not "
                               "an HBM bound)", 10, SWEEP_RADII, 1)
        # the mode that is bit-exact over all 10 iterations (C3's parity bar:
        # tests/test_configs_gpu.py::test_c3_full_exact_bit_exact)
        subs["C3_exact"] = sub_sweep(ctx, c3, "C3: 4096^2 uint8, 10 exact iterations per "
                                     "radius (bit-identical to the reference at every "
                                     "iteration)", 10, SWEEP_RADII, 1, reps=3, mode="exact")
        result["sub"] = subs

    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        if x_host is None:
            x_host = x.cpu()
        result["cpu_baseline"] = cpu_baseline_c5(x_host.numpy(), r)
    if rank == 0:
        print(json.dumps(result), flush=True)


# ---- C1..C4 -------------------------------------------------------------------

def run_batch(args, world, rank, local):
    """C1..C4: each rank filters its own full batch (weak scaling)."""
    import ctypes

    import torch

    import paper_2108_05021_b200 as ob
    from paper_2108_05021_b200 import synth

    torch.cuda.set_device(local)
    cfg = synth.CONFIGS[args.workload]
    r = args.radius or cfg.radius
    iters = args.iterations or cfg.iterations
    x = synth.make_input(args.workload)  # (B, H, W), seeded, identical on every rank
    B, H, W = x.shape
    px = B * H * W
    ctx = ob.Context(local)
    d_in = torch.from_numpy(x).cuda()
    d_out = torch.empty((B, H, W), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    run = lambda: ctx.iterate(d_in, r, iters, mode=args.mode, out=d_out)  # noqa: E731
    for _ in range(max(args.warmup, 0)):
        run()
    torch.cuda.synchronize()
    kernel = ctx.last_kernel
    clocks = ClockSampler(local)
    launches0 = ctx.launches
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    ms = time_steps(run, args.steps, stream, pre=lambda i: flush.fill_(i & 0xFF))
    barrier(world)
    clk = clocks.stop()
    launches = int(allreduce(ctx.launches - launches0, world, "sum"))
    total_ms = allreduce(sum(ms), world, "max")
    value = world * px * iters * args.steps / (total_ms / 1000.0) / 1e6
    in_b = IN_BYTES[cfg.dtype]
    alg = px * ((in_b + 8) + (iters - 1) * 16) / iters
    result = {
        "metric": METRIC, "value": round(value, 3), "unit": "Mpx-iter/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(total_ms / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(cfg, r, iters), "batch_per_gpu": B, "height": H,
                   "width": W, "radius": r, "iterations": iters, "mode": args.mode,
                   "storage": "f64 between passes (input dtype on the first pass)",
                   "l2": "L2 flushed (256 MiB write) between timed steps",
                   "parallelism": f"batch-sharded dp{world} (each rank its own {B}-plane batch)"},
        "roofline": roofline(alg, sum(ms) / (args.steps * iters), kernel, args.workload,
                             args.mode, f"read U^t + write U^{{t+1}}: first pass {in_b}+8 B, "
                             "then 8+8 B; avg launch = step time / iterations"),
        "gpu_launches": launches,
        "launches_per_pass": round(launches / max(1, args.steps * iters * world), 3),
        "clocks": clk,
    }
    if not args.no_e2e:
        h_in = torch.from_numpy(x).pin_memory()
        h_out = torch.empty((B, H, W), dtype=torch.float64).pin_memory()
        lib = ctx._lib
        code = {"u8": 0, "f32": 1, "f64": 2}[cfg.dtype]
        mcode = {"exact": 0, "fast": 1}[args.mode]

        def e2e_call():
            st = lib.osbf_gpu_osbf_host(ctx.handle, code, ctypes.c_void_p(h_in.data_ptr()),
                                        ctypes.c_void_p(h_out.data_ptr()), W, H, B, r, iters,
                                        mcode)
            if st != 0:
                raise RuntimeError(lib.osbf_gpu_last_error().decode())

        e2e_call()
        e2e_steps = max(1, min(args.steps, 5))
        barrier(world)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            e2e_call()
        dt = allreduce(time.perf_counter() - t0, world, "max")
        result["e2e"] = {"value": round(world * px * iters * e2e_steps / dt / 1e6, 3),
                         "unit": "Mpx-iter/s",
                         "h2d_bytes_per_step": int(h_in.numel() * h_in.element_size()),
                         "d2h_bytes_per_step": int(h_out.numel() * 8), "steps": e2e_steps,
                         "api": "osbf_gpu_osbf_host (C ABI, pinned host buffers)",
                         "matches_device_path": bool(torch.equal(
                             h_out.view(torch.int64), d_out.cpu().view(torch.int64)))}
    if world == 1 and rank == 0 and not args.no_cpu_baseline:
        import numpy as np

        planes = x.reshape(-1, H, W)
        threads = os.cpu_count() or 1
        v, kind, t = cpu_rate(np.asarray(planes[0]), r, threads)
        v1, _, t1 = cpu_rate(np.asarray(planes[0][: max(64, H // 4)]), r, 1)
        result["cpu_baseline"] = {
            "value": round(v, 3), "unit": "Mpx-iter/s", "cores": threads, "kind": kind,
            "sample": f"reference osbf::osbf, 1 pass over one {H}x{W} plane, median of 3 "
                      f"({t:.3f} s), {threads} threads",
            "one_thread": {"value": round(v1, 3), "cores": 1,
                           "sample": f"1 pass over {max(64, H // 4)} rows, median of 3"},
            "cpu_model": cpu_model()}
    if rank == 0:
        print(json.dumps(result), flush=True)
    ctx.close()


def main():
    args = parse()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    elif args.workload == "C5":
        run_c5(args, world, rank, local)
    else:
        run_batch(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
