#!/usr/bin/env python
"""Benchmark of the SPCN hot path on B200 (contract: one JSON line on rank 0).

Workload (BASELINE.json configs[3], the north-star case): a synthetic
100000 x 100000 (10 Gpixel) H&E whole-slide image, rendered on the GPU
(model of src/synthetic.py), sharded into equal row bands across N GPUs
(strong scaling: total work fixed).  One step = ``fit`` of the source slide
(seeded patch sampling → i0 → sparse-NMF basis → density p99, all on the
device) + ``transform`` of every pixel against a fixed target profile (the
target is fitted once before timing, as with a --profile target).  Input and
output (30 GB each) stay resident in HBM; they are >> the 126 MB L2, so no
flush is needed between steps.

    python bench.py                          # N=1, defaults
    python bench.py --impl reference         # the reference's CPU path (oracle port)
    torchrun --nproc-per-node N bench.py --gpus N

Extra keys: roofline (dominant kernel = the
fused recolor launch, 6 algorithmic bytes/pixel), cpu_baseline (oracle port
on the host cores, bounded sample, extrapolated), e2e (public API with
pinned host buffers, H2D+D2H inside the timed region), gpu_launches,
clocks (NVML sampled during the timed region).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixels/sec normalized (whole box, 1/2/4/8 B200) + % of HBM/MUFU roofline"
BYTES_PER_PX = 6          # pass 2: 3 read + 3 write


def parse():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--width", type=int, default=100_000)
    ap.add_argument("--height", type=int, default=100_000)
    ap.add_argument("--tissue", type=float, default=0.6)
    ap.add_argument("--layout", default="scatter")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--precision", default="exact", choices=("exact", "fast", "strict"))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--e2e-workers", type=int, default=3, help="CUDA streams of the host transform")
    ap.add_argument("--cpu-rows", type=int, default=0,
                    help="rows of the CPU-baseline band (default: 4 strips of 64 rows per core)")
    ap.add_argument("--dist-backend", choices=("nccl", "gloo"), default="nccl",
                    help="gloo: functional check of the N>1 path on one GPU (not a measurement)")
    ap.add_argument("--no-global-line", action="store_true",
                    help="wsi: skip the extra global-p99 measurement")
    ap.add_argument("--p99-mode", choices=("sample", "global"), default="sample",
                    help="sample = reference semantics (default); global = whole-slide p99 passes")
    ap.add_argument("--workload", choices=("wsi", "batch", "tile"), default="wsi",
                    help="wsi = configs[3] (default); batch = configs[1] (4096 x 512^2 "
                         "patches); tile = configs[0] (2048^2 tile vs 2048^2 target)")
    ap.add_argument("--batch", type=int, default=4096)
    ap.add_argument("--patch", type=int, default=512)
    ap.add_argument("--batch-chunk", type=int, default=256,
                    help="items per pipelined chunk of the host-batch e2e leg")
    ap.add_argument("--cpu-patches", type=int, default=max(8, os.cpu_count() or 1),
                    help="patches in the CPU-baseline sample (one per host core)")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
_REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
            0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown"}


def _clock_loop(index, period, halt, q):
    """NVML sampling loop (child process: never starved by the parent's GIL)."""
    samples, reasons, max_mhz = [], set(), None
    try:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        while not halt.is_set():
            samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
            mask = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
            for bit, name in _REASONS.items():
                if mask & bit:
                    reasons.add(name)
            time.sleep(period)
    except Exception as exc:  # pragma: no cover - NVML missing
        reasons.add(f"nvml-unavailable: {exc}")
    q.put((samples, sorted(reasons), max_mhz))


class Clocks:
    """NVML sampler (SM clock, throttle reasons) over the timed region, in a
    forked child process sampling every `period` seconds."""

    def __init__(self, index: int, period: float = 0.005):
        import multiprocessing as mp

        self.index, self.period = index, period
        self._ctx = mp.get_context("fork")
        self._halt, self._q, self._p = self._ctx.Event(), self._ctx.Queue(), None

    def start(self):
        self._p = self._ctx.Process(target=_clock_loop,
                                    args=(self.index, self.period, self._halt, self._q),
                                    daemon=True)
        self._p.start()

    def stop(self):
        self._halt.set()
        try:
            samples, reasons, max_mhz = self._q.get(timeout=10)
        except Exception:  # pragma: no cover
            samples, reasons, max_mhz = [], ["sampler-lost"], None
        self._p.join(timeout=5)
        return {"sm_mhz": float(statistics.median(samples)) if samples else None,
                "sm_max_mhz": max_mhz, "reasons": reasons, "samples": len(samples)}


# --------------------------------------------------------------------------- distributed
def dist_setup(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch

    if world > 1:
        local = local % max(1, torch.cuda.device_count())   # gloo checks may share one GPU
        torch.cuda.set_device(local)
        import torch.distributed as dist

        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:   # code-path check only (host-staged collectives); never for timing
            dist.init_process_group("gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return rank, world, local


def _max_over_ranks(x: float, dev) -> float:
    """Max of a host scalar over ranks (device tensor under NCCL, host under gloo)."""
    import torch
    import torch.distributed as dist

    on = dev if dist.get_backend() == "nccl" else torch.device("cpu")
    tt = torch.tensor([x], device=on, dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return float(tt.item())


def band_of(height, rank, world):
    per = height // world
    r0 = rank * per
    rows = per if rank < world - 1 else height - r0
    return r0, rows


# --------------------------------------------------------------------------- CPU baseline
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def cpu_band_rows(cores: int, strip: int = 64, per_core: int = 4) -> int:
    """Rows of the CPU-baseline band: per_core strips of `strip` rows per host
    core, so every worker of the reference's pool stays busy (src/pipeline.py
    :311-315 keeps at most `workers` strips in flight)."""
    return per_core * cores * strip


def cpu_reference_run(band: np.ndarray, target: dict, cores: int, strips=(64,)):
    """Time the reference algorithm (oracle port) on a host band: one fit, then
    one transform per strip height.  Returns (t_fit, {strip: t_transform})."""
    from oracle import spcn_oracle as orc

    t0 = time.perf_counter()
    fp = orc.fit_params(band)
    t_fit = time.perf_counter() - t0
    t_x = {}
    for sh in strips:
        t1 = time.perf_counter()
        orc.run_transform(band, fp, target, strip_height=sh, workers=cores)
        t_x[sh] = time.perf_counter() - t1
    return t_fit, t_x


def extrapolated_mpx(total_px, band_px, t_fit, t_x):
    """Whole-slide Mpx/s from a band: one fit + linear-in-pixels transform
    (linearity: criterion 10, tests/test_acceptance.py:286-289)."""
    return total_px / (t_fit + t_x * total_px / band_px) / 1e6


def cpu_sample_desc(rows, width, cores, t_fit, t_x, total):
    band_px = rows * width
    parts = ", ".join(f"strip {sh}: {band_px / t / 1e6:.1f} Mpx/s ({t:.2f} s, "
                      f"{-(-rows // sh)} strips)" for sh, t in sorted(t_x.items()))
    return (f"{rows} x {width} band ({band_px / 1e6:.0f} Mpx) of the same synthetic model, "
            f"reference algorithm (oracle port, NumPy) on {cores} threads of "
            f"'{cpu_model()}': fit {t_fit:.3f} s; transform {parts}; value = one fit + the "
            f"strip-64 transform (the faster CPU setting) extrapolated linearly in pixels "
            f"(criterion 10) to the whole {total / 1e9:.2f} Gpx: "
            f"{t_fit + t_x[64] * total / band_px:.0f} s")


# --------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The reference's CPU path on the box's host cores: each step = fit + transform
    (strip 64, all cores) of a bounded band of the workload (4 strips per core);
    one extra strip-1024 transform (the reference default) is reported beside it."""
    if rank != 0:
        return 0
    from oracle import spcn_oracle as orc

    cores = os.cpu_count() or 1
    rows = min(args.height, max(64, args.cpu_rows or cpu_band_rows(cores)))
    band = orc.render_band(args.width, args.height, args.seed, rows, tissue_fraction=args.tissue,
                           layout=args.layout)
    tgt_px, _, _ = orc.render(1024, 1024, args.seed + 1, tissue_fraction=0.6)
    target = orc.fit_params(tgt_px)
    total = args.width * args.height
    if args.warmup:            # warm thread pools / allocator on a small piece
        cpu_reference_run(band[:min(rows, 4 * 64)], target, cores)
    steps = max(1, min(args.steps, 2))
    times = []
    for _ in range(steps):
        tf, tx = cpu_reference_run(band, target, cores)
        times.append(tf + tx[64])
    _, tx1024 = cpu_reference_run(band, target, cores, strips=(1024,))
    sec = statistics.median(times)
    band_px = rows * args.width
    value = extrapolated_mpx(total, band_px, tf, tx[64])
    sample = cpu_sample_desc(rows, args.width, cores, tf, {64: tx[64], 1024: tx1024[1024]},
                             total)
    line = {"metric": METRIC, "value": round(value, 3), "unit": "Mpx/s", "n_gpus": world,
            "steps": steps, "warmup": 1 if args.warmup else 0, "ms_per_step": round(sec * 1e3, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": workload_config(args, world),
            "cpu_baseline": {"value": round(value, 3), "unit": "Mpx/s", "cores": cores,
                             "kind": "port", "cpu": cpu_model(), "sample": sample,
                             "strip1024_value": round(extrapolated_mpx(total, band_px, tf,
                                                                       tx1024[1024]), 3)},
            "e2e": {"value": round(value, 3), "unit": "Mpx/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(args, world):
    npx = args.width * args.height
    tag = ("C3" if npx == 20000 * 20000 else
           "C5" if args.tissue <= 0.35 else "C4" if npx == 100000 * 100000 else "WSI")
    return {"workload": f"{tag}: {args.width}x{args.height} synthetic H&E WSI "
                        f"({npx / 1e9:.2f} Gpx, tissue {args.tissue} "
                        f"{args.layout}); step = fit(source) + transform(all pixels) vs a "
                        "fixed target profile",
            "width": args.width, "height": args.height, "precision": args.precision,
            "parallelism": f"row-band x{world}", "p99_mode": args.p99_mode,
            "l2": f"input+output {6 * npx / 1e9:.1f} GB per step >> 126 MB L2 (no flush needed)"}


# --------------------------------------------------------------------------- batch (configs[1])
def batch_config(args, world):
    return {"workload": f"C2: batch of {args.batch} synthetic {args.patch}x{args.patch} H&E "
                        "patches (8 groups of tissue fraction / background), each fitted and "
                        "normalized against one fixed target profile; step = "
                        "normalize_batch(all patches)",
            "batch": args.batch, "patch": args.patch, "precision": args.precision,
            "parallelism": f"independent batches x{world}",
            "l2": f"input+output {2 * 3 * args.batch * args.patch ** 2 / 1e9:.1f} GB per step "
                  ">> 126 MB L2 (no flush needed)"}


def _batch_images(args, seed, n, dev):
    import torch

    from paper_1901_03088_b200 import synthetic

    P = args.patch
    imgs = torch.empty((n, P, P, 3), dtype=torch.uint8, device=dev)
    groups = 8
    per = -(-n // groups)
    for g in range(groups):
        a, b = g * per, min(n, (g + 1) * per)
        if a >= b:
            break
        i0 = (255 - 3 * g, 252 - 2 * g, 255 - g)
        synthetic.render_rows(imgs[a:b].view(-1), P, (b - a) * P, 0, (b - a) * P, seed + 97 * g,
                              i0=i0, tissue_fraction=0.3 + 0.08 * g, dense=bool(g & 1))
    return imgs


def run_batch(args, rank, world, local):
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import _lib, synthetic

    dev = torch.device("cuda", local if world > 1 else 0)
    n, P = args.batch, args.patch
    imgs = _batch_images(args, args.seed + 1000 * rank, n, dev)
    out = torch.empty_like(imgs)
    tgt = synthetic.render_slide(2048, 2048, args.seed + 1, tissue_fraction=0.6)
    target = pb.fit(pb.DeviceSource(tgt))
    del tgt
    xform_ms = []

    def step(record=False):
        fits = pb.fit_batch(imgs)
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        _, errors = pb.transform_batch(imgs, fits, target, out, precision=args.precision)
        if record:
            e1.record()
            xform_ms.append((e0, e1))
        return errors

    for _ in range(args.warmup):
        errors = step()
    failed = sum(e is not None for e in errors)
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = Clocks(dev.index if dev.index is not None else 0)
    clocks.start()
    time.sleep(0.05)
    L = _lib.lib()
    launches0 = L.spcn_launch_count()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step(record=True)
    t1.record()
    torch.cuda.synchronize()
    launches = L.spcn_launch_count() - launches0
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    npx = n * P * P
    value = npx * world / (ms * 1e-3) / 1e6
    x_ms = statistics.mean(a.elapsed_time(b) for a, b in xform_ms)
    achieved = BYTES_PER_PX * npx / (x_ms * 1e-3) / 1e9
    peak, peak_src = _hbm_peak()
    line = {"metric": METRIC, "value": round(value, 3), "unit": "Mpx/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype_label(args.precision),
            "data": "synthetic (on-GPU generator, model of src/synthetic.py)",
            "config": batch_config(args, world),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "spcn_xform_batch (k_xform_batch + k_repair_batch)",
                         "kernel_ms": round(x_ms, 4), "share_of_step": round(x_ms / ms, 4),
                         "algorithmic_bytes_per_px": BYTES_PER_PX, "peak_source": peak_src,
                         "mufu": mufu_roofline(npx, x_ms, clk)},
            "gpu_launches": int(launches), "clocks": clk, "failed_items": failed}
    if not args.no_e2e:
        h_in = torch.empty(imgs.shape, dtype=torch.uint8, pin_memory=True)
        h_in.copy_(imgs)
        h_out = torch.empty_like(h_in).pin_memory()
        times = []
        for i in range(args.e2e_steps + 1):
            torch.cuda.synchronize()
            t_a = time.perf_counter()
            pb.normalize_batch_host(h_in, target, h_out, chunk=args.batch_chunk, streams=6,
                                    precision=args.precision)
            torch.cuda.synchronize()
            if i:
                times.append(time.perf_counter() - t_a)
        sec = min(times)
        line["e2e"] = {"value": round(npx * world / sec / 1e6, 3), "unit": "Mpx/s",
                       "h2d_bytes_per_step": 3 * npx, "d2h_bytes_per_step": 3 * npx,
                       "seconds_per_step": round(sec, 4),
                       "path": f"pb.normalize_batch_host(pinned host batch -> pinned host), "
                               f"{args.batch_chunk}-item chunks pipelined over 6 streams"}
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_batch_baseline(args, imgs, target)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def _cpu_patch_run(px, target):
    from oracle import spcn_oracle as orc

    fp = orc.fit_params(px)
    return orc.run_transform(px, fp, target, strip_height=1024, workers=1)


def cpu_batch_baseline(args, imgs, target, cores=None):
    """Oracle port on a bounded number of patches, one patch per host core
    (the reference's cmd_batch runs patches one after another; src/cli.py:270-301)."""
    from concurrent.futures import ThreadPoolExecutor

    cores = cores or (os.cpu_count() or 1)
    k = max(1, min(args.cpu_patches, imgs.shape[0]))
    stride = max(1, imgs.shape[0] // k)
    sample = [imgs[i * stride].cpu().numpy() for i in range(k)]
    tgt = dict(i0=np.asarray(target.i0), basis=np.asarray(target.basis),
               p99=np.asarray(target.stats.p99))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(cores, k)) as pool:
        list(pool.map(lambda p: _cpu_patch_run(p, tgt), sample))
    sec = time.perf_counter() - t0
    v = k * args.patch ** 2 / sec / 1e6
    return {"value": round(v, 3), "unit": "Mpx/s", "cores": min(cores, k), "kind": "port",
            "sample": f"{k} of the {imgs.shape[0]} patches (every {stride}th), fit + transform "
                      f"each with the oracle port, {min(cores, k)} patches in parallel; "
                      f"{sec:.2f} s"}


def mufu_roofline(npx, kernel_ms, clk):
    """Second roofline of the recolour: 3 MUFU.EX2 per pixel vs
    148 SM x 16 MUFU/clk at the SM clock measured during the timed region."""
    import torch

    mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    peak = sms * 16 * mhz * 1e6
    achieved = 3.0 * npx / (kernel_ms * 1e-3)
    return {"ops_per_px": 3, "achieved_gops": round(achieved / 1e9, 1),
            "peak_gops": round(peak / 1e9, 1), "frac": round(achieved / peak, 4),
            "peak_source": f"{sms} SM x 16/clk x {mhz:.0f} MHz (measured clock)"}


def dtype_label(precision: str) -> str:
    """What the path computes in: EXACT = fp32 arithmetic certified per pixel,
    fp64 (reference operation order) for the uncertified ones — output bytes
    identical to the fp64 reference; STRICT = fp64 throughout; FAST = fp32."""
    return {"exact": "f64-exact (fp32 certified + fp64 repair; u8 out byte-identical)",
            "strict": "f64", "fast": "f32 (+-1 LSB)"}[precision]


def _hbm_peak():
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        peaks = {}
    if "hbm_gbs" in peaks:
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# --------------------------------------------------------------------------- tile (configs[0])
def run_tile(args, rank, world, local):
    """C1: one 2048^2 tile normalized to a 2048^2 target — pb.normalize (fit
    source + fit target + transform), the reference's _normalize_one."""
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import _lib, synthetic

    side = 2048
    dev = torch.device("cuda", local if world > 1 else 0)
    src = synthetic.render_slide(side, side, args.seed + 10 * rank, tissue_fraction=0.6)
    tgt = synthetic.render_slide(side, side, args.seed + 1, tissue_fraction=0.6)
    for _ in range(args.warmup):
        pb.normalize(src, tgt, precision=args.precision, p99_mode=args.p99_mode)
    torch.cuda.synchronize()
    L = _lib.lib()
    launches0 = L.spcn_launch_count()
    clocks = Clocks(dev.index if dev.index is not None else 0)
    clocks.start()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        pb.normalize(src, tgt, precision=args.precision, p99_mode=args.p99_mode)
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = L.spcn_launch_count() - launches0
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    npx = side * side
    line = {"metric": METRIC, "value": round(npx * world / (ms * 1e-3) / 1e6, 3), "unit": "Mpx/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": dtype_label(args.precision),
            "data": "synthetic (on-GPU generator, model of src/synthetic.py)",
            "config": {"workload": "C1: 2048x2048 tile normalized to a 2048x2048 target "
                                   "(fit both + transform, reference defaults)",
                       "precision": args.precision, "p99_mode": args.p99_mode,
                       "l2": "per-step working set 25 MB fits L2 (fit-dominated step)"},
            "gpu_launches": int(launches), "clocks": clk}
    if not args.no_e2e:
        s_np, t_np = src.cpu().numpy(), tgt.cpu().numpy()
        times = []
        for i in range(args.e2e_steps + 1):
            a = time.perf_counter()
            pb.normalize(s_np, t_np, precision=args.precision, p99_mode=args.p99_mode)
            if i:
                times.append(time.perf_counter() - a)
        sec = min(times)
        line["e2e"] = {"value": round(npx * world / sec / 1e6, 3), "unit": "Mpx/s",
                       "h2d_bytes_per_step": 2 * 3 * npx, "d2h_bytes_per_step": 3 * npx,
                       "seconds_per_step": round(sec, 4),
                       "path": "pb.normalize(numpy source, numpy target) -> numpy"}
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import spcn_oracle as orc

        s_np, t_np = src.cpu().numpy(), tgt.cpu().numpy()
        a = time.perf_counter()
        fs, ft = orc.fit_params(s_np), orc.fit_params(t_np)
        orc.run_transform(s_np, fs, ft, strip_height=64, workers=os.cpu_count() or 1)
        sec = time.perf_counter() - a
        line["cpu_baseline"] = {"value": round(npx / sec / 1e6, 3), "unit": "Mpx/s",
                                "cores": os.cpu_count() or 1, "kind": "port",
                                "sample": f"the whole C1 step (fit source + fit target + "
                                          f"transform, strip 64) with the oracle port: {sec:.2f} s"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


# --------------------------------------------------------------------------- our arm
def run_ours(args, rank, world, local):
    import torch

    import paper_1901_03088_b200 as pb
    from paper_1901_03088_b200 import _lib, synthetic

    dev = torch.device("cuda", local if world > 1 else 0)
    r0, rows = band_of(args.height, rank, world)
    W = args.width
    slide = torch.empty((rows, W, 3), dtype=torch.uint8, device=dev)
    synthetic.render_rows(slide, W, args.height, r0, rows, args.seed, tissue_fraction=args.tissue,
                          layout=args.layout)
    out = torch.empty_like(slide)
    tgt = synthetic.render_slide(2048, 2048, args.seed + 1, tissue_fraction=0.6)
    target = pb.fit(pb.DeviceSource(tgt))
    del tgt
    src = pb.DeviceSource(slide)
    group = None
    if world > 1:
        from paper_1901_03088_b200 import distributed

        group = distributed.RowBandGroup(args.width, args.height, r0, rows)

    xform_ms = []
    # one GPU, pooled p99, EXACT: the drop-in normalize() runs fit -> transform
    # with the recolouring built on the device (no host round trip between)
    args.fused = os.environ.get("SPCN_FUSED", "1") != "0"

    def fused_step():
        return args.fused and args.p99_mode == "sample" and args.precision == "exact"

    def step(record=False):
        if fused_step():
            if group is None:
                return pb.normalize(slide, target, out=out)
            return group.fit_transform(src, target, out)
        if group is None:
            fp = pb.fit(src, p99_mode=args.p99_mode)
        else:
            fp = group.fit(src, p99_mode=args.p99_mode)
        sink = pb.DeviceWriter(W, rows, out=out)
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        if group is None:
            pb.transform(src, fp, target, sink, precision=args.precision)
        else:   # calibration split across the ranks (one max all-reduce)
            group.transform(src, fp, target, sink, precision=args.precision)
        if record:
            e1.record()
            xform_ms.append((e0, e1))
        return fp

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = Clocks(dev.index if dev.index is not None else 0)
    clocks.start()
    time.sleep(0.05)
    L = _lib.lib()
    launches0 = L.spcn_launch_count()
    torch.cuda.synchronize()
    import ctypes

    n_k, k_tot = ctypes.c_int64(0), ctypes.c_double(0.0)
    L.spcn_xform_timing(ctypes.byref(n_k), ctypes.byref(k_tot))     # clear
    L.spcn_xform_timing_enable(1)
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(args.steps):
        step(record=True)
    t1.record()
    torch.cuda.synchronize()
    L.spcn_xform_timing_enable(0)
    _lib.check(L.spcn_xform_timing(ctypes.byref(n_k), ctypes.byref(k_tot)), "xform_timing")
    launches = L.spcn_launch_count() - launches0
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / args.steps
    if world > 1:
        ms = _max_over_ranks(ms, dev)
    total = args.width * args.height
    value = total / (ms * 1e-3) / 1e6
    call_ms = statistics.mean(a.elapsed_time(b) for a, b in xform_ms) if xform_ms else None
    npx_rank = rows * W
    # the dominant kernel alone: k_xform_warp's launches timed with CUDA
    # events on their stream inside the timed region (spcn_xform_timing)
    x_ms = k_tot.value / max(1, n_k.value) if n_k.value else call_ms
    achieved = BYTES_PER_PX * npx_rank / (x_ms * 1e-3) / 1e9
    peaks = {}
    try:
        peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        pass
    peak = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "measured" if "hbm_gbs" in peaks else "fallback"
    traffic, traffic_px = None, None
    try:
        prof = json.load(open(os.path.join(ROOT, "profiles", "xform_traffic.json")))
        traffic_px = float(prof["bytes_per_px"])
        traffic = round(traffic_px * npx_rank)       # DRAM bytes per launch (ncu, scaled)
    except Exception:
        pass

    line = {"metric": METRIC, "value": round(value, 3), "unit": "Mpx/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": dtype_label(args.precision),
            "data": "synthetic (on-GPU generator, model of src/synthetic.py)",
            "config": workload_config(args, world),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "traffic": traffic, "traffic_bytes_per_px": traffic_px,
                         "traffic_source": "profiles/xform_traffic.json (ncu --set full)",
                         "kernel": ("k_xform_warp_c (main recolour launch of the device-built "
                                    "recolouring, spcn_xform_rgb8_fitted / _run)"
                                    if fused_step() else
                                    "k_xform_warp (main recolour launch of spcn_xform_rgb8)"),
                         "kernel_ms": round(x_ms, 4), "kernel_launches_timed": int(n_k.value),
                         "share_of_step": round(x_ms / ms, 4),
                         "transform_call_ms": round(call_ms, 4) if call_ms else None,
                         "transform_call_frac": round(BYTES_PER_PX * npx_rank / (call_ms * 1e-3)
                                                      / 1e9 / peak, 4) if call_ms else None,
                         "algorithmic_bytes_per_px": BYTES_PER_PX,
                         "peak_source": f"{peak_src} (MEASURED_PEAKS.json hbm_gbs)",
                         "mufu": mufu_roofline(npx_rank, x_ms, clk)},
            "gpu_launches": int(launches), "clocks": clk}

    # ---- variants of the same step, a few steps each, same timing rules
    def alt_steps(attr, value):
        old = getattr(args, attr)
        setattr(args, attr, value)
        try:
            n_alt = max(3, args.steps // 5)
            step()
            torch.cuda.synchronize()
            if world > 1:
                torch.distributed.barrier()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for _ in range(n_alt):
                step()
            g1.record()
            torch.cuda.synchronize()
            gms = g0.elapsed_time(g1) / n_alt
            if world > 1:
                gms = _max_over_ranks(gms, dev)
            return {"value": round(total / (gms * 1e-3) / 1e6, 3), "unit": "Mpx/s",
                    "ms_per_step": round(gms, 4), "steps": n_alt, "warmup": 1}
        finally:
            setattr(args, attr, old)

    if not args.no_global_line:
        if args.p99_mode == "sample":
            # whole-slide percentiles (configs[3]: the colour-count table
            # all-reduced across the row bands)
            line["global_p99_mode"] = dict(alt_steps("p99_mode", "global"), note=(
                "same step with fit(p99_mode='global'): exact p99 of every non-white pixel "
                "(one k_stats_cube pass into per-rank colour tables; "
                + ("a 64 KiB entry-histogram all-reduce + a small all-gather over NCCL"
                   if world > 1 else "selection on this rank") + ")"))
        if args.p99_mode == "sample" and args.precision == "exact" and args.fused:
            line["host_params_step"] = dict(alt_steps("fused", False), note=(
                "same step as fit + transform (pb.*, or RowBandGroup.* at N > 1): the "
                "recolouring's parameters built on the host between the fit's read-back "
                "and the transform launch"))
        if args.precision == "exact":
            # the north star's stated tolerance (+-1 LSB on >= 99.9 % of pixels)
            line["fast_precision"] = dict(alt_steps("precision", "fast"), note=(
                "same step with precision='fast' (no certification/repair; within +-1 LSB of "
                "the reference on >= 99.9 % of pixels, tests/test_xform_gpu.py); the headline "
                "value is the byte-exact mode"))
    # ---- end-to-end through the public API with pinned host buffers
    if not args.no_e2e:
        try:
            line["e2e"] = e2e(args, pb, slide, target, rank, world, group)
        except Exception as exc:  # pragma: no cover
            line["e2e"] = {"value": None, "unit": "Mpx/s", "error": repr(exc)[:200]}
    # ---- CPU baseline (rank 0, N = 1 only)
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            line["cpu_baseline"] = cpu_baseline(args, slide, target)
        except Exception as exc:  # pragma: no cover
            line["cpu_baseline"] = {"value": None, "error": repr(exc)[:200]}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def e2e(args, pb, slide, target, rank, world, group=None):
    """Same metric through pb.fit/pb.transform with host (pinned) input and output.
    N > 1: the whole slide's fit is a collective over the row bands
    (RowBandGroup), which reads resident bands, so each rank uploads its band
    (pinned, timed), runs RowBandGroup.fit_transform and downloads its band
    (timed) — the same bytes as the device step."""
    import torch

    if world > 1 and group is not None:
        return _e2e_group(args, pb, slide, target, group, world)

    rows, W = slide.shape[0], slide.shape[1]
    nbytes = slide.numel()
    avail = 0
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable"):
                avail = int(ln.split()[1]) * 1024
    except Exception:
        pass
    use_rows = rows
    if avail and 2.3 * nbytes > avail / max(1, world):
        use_rows = max(1024, int(rows * (avail / max(1, world)) / (2.5 * nbytes)))
    h_src = torch.empty((use_rows, W, 3), dtype=torch.uint8, pin_memory=True)
    h_src.copy_(slide[:use_rows])
    h_dst = torch.empty_like(h_src).pin_memory()
    src = pb.ArraySource(h_src.numpy())
    times, fit_s = [], []
    for i in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fp = pb.fit(src)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        sink = pb.ArrayWriter(W, use_rows, out=h_dst.numpy())
        pb.transform(src, fp, target, sink, precision=args.precision, workers=args.e2e_workers)
        torch.cuda.synchronize()
        if i:                       # first run = warm-up
            times.append(time.perf_counter() - t0)
            fit_s.append(t1 - t0)
    sec = min(times)
    if world > 1:
        sec = _max_over_ranks(sec, torch.device("cuda", torch.cuda.current_device()))
    px = use_rows * W * world
    res = {"value": round(px / sec / 1e6, 3), "unit": "Mpx/s",
           "h2d_bytes_per_step": int(use_rows * W * 3), "d2h_bytes_per_step": int(use_rows * W * 3),
           "rows_per_gpu": use_rows, "seconds_per_step": round(sec, 4),
           "fit_seconds": round(min(fit_s), 4),
           "path": f"pb.fit(ArraySource(pinned)) + pb.transform(-> ArrayWriter(pinned)), "
                   f"{args.e2e_workers} streams"}
    del h_src, h_dst
    return res


def _e2e_group(args, pb, slide, target, group, world):
    import torch

    rows, W = slide.shape[0], slide.shape[1]
    h_src = torch.empty((rows, W, 3), dtype=torch.uint8, pin_memory=True)
    h_src.copy_(slide)
    h_dst = torch.empty_like(h_src).pin_memory()
    d_src = torch.empty_like(slide)
    d_dst = torch.empty_like(slide)
    dev = slide.device
    times = []
    for i in range(args.e2e_steps + 1):
        torch.cuda.synchronize()
        torch.distributed.barrier()
        t0 = time.perf_counter()
        d_src.copy_(h_src, non_blocking=True)
        group.fit_transform(pb.DeviceSource(d_src), target, d_dst)
        h_dst.copy_(d_dst, non_blocking=True)
        torch.cuda.synchronize()
        if i:
            times.append(time.perf_counter() - t0)
    sec = _max_over_ranks(min(times), dev)
    res = {"value": round(rows * W * world / sec / 1e6, 3), "unit": "Mpx/s",
           "h2d_bytes_per_step": int(rows * W * 3), "d2h_bytes_per_step": int(rows * W * 3),
           "rows_per_gpu": rows, "seconds_per_step": round(sec, 4),
           "path": "per rank: band H2D (pinned) -> RowBandGroup.fit_transform -> band D2H "
                   "(pinned); max over ranks"}
    del h_src, h_dst, d_src, d_dst
    return res


def cpu_baseline(args, slide, target):
    """Oracle port of the reference path on the host cores (bounded band of the
    same slide, 4 strips of 64 rows per core), strip heights 64 and 1024."""
    cores = os.cpu_count() or 1
    rows = min(slide.shape[0], max(64, args.cpu_rows or cpu_band_rows(cores)))
    band = slide[:rows].cpu().numpy()
    tgt = dict(i0=np.asarray(target.i0), basis=np.asarray(target.basis),
               p99=np.asarray(target.stats.p99))
    tf, tx = cpu_reference_run(band, tgt, cores, strips=(64, 1024))
    band_px = rows * args.width
    total = args.width * args.height
    return {"value": round(extrapolated_mpx(total, band_px, tf, tx[64]), 3), "unit": "Mpx/s",
            "cores": cores, "kind": "port", "cpu": cpu_model(),
            "strip1024_value": round(extrapolated_mpx(total, band_px, tf, tx[1024]), 3),
            "sample": cpu_sample_desc(rows, args.width, cores, tf, tx, total)}


def _free_port() -> int:
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def launch_ranks(args) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run on 127.0.0.1, with NCCL's communicator logging on
    (stderr); rank 0 prints the JSON line.  Exit code = the launcher's."""
    import subprocess

    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


def check_world(args, world: int) -> None:
    """--gpus must match the launched world (never measure N=1 under an N-GPU
    command); the NCCL arm needs one GPU per rank."""
    if args.gpus != world:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "ours" and world > 1 and args.dist_backend == "nccl":
        import torch

        if torch.cuda.device_count() < world:
            raise SystemExit(f"bench.py: --gpus {world} needs {world} GPUs, "
                             f"{torch.cuda.device_count()} visible")


def main():
    args = parse()
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1 and args.impl == "ours":
        return launch_ranks(args)
    if world_env is not None or args.impl == "ours":
        check_world(args, int(world_env or "1"))
    rank, world, local = dist_setup(args) if args.impl == "ours" else (
        int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    if args.workload == "batch":
        return run_batch(args, rank, world, local)
    if args.workload == "tile":
        return run_tile(args, rank, world, local)
    return run_ours(args, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
