#!/usr/bin/env python
"""FNR filter benchmark: Mpix/s filtered (detect+median) on B200, BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl b200|reference]

One "step" is one filter pass (method "fnr", passes=1 — the run_filter default,
filters.py:83) over the BASELINE workload. BASELINE.json's metric names no config, so
the default workload is the largest single-GPU config, c5 (4096 x 640x480 u8 video
frames, 3x3 window); `--config c1..c4` selects another one.

Multi-GPU (torchrun, one rank per GPU): the BASELINE workload is SPLIT
across the ranks — c2 / c3 / c5 by frames (B/N contiguous frames per rank, the
reference's band bounds), c4 by row strips (8192/N rows plus an r-row halo on each side,
clamped against the global frame through irdn_filter_strip_*), strong scaling; c1 (one
512x512 frame) runs as replicas (weak scaling). No data-path collective: the filter
shards are independent; outputs stay sharded, and one gather of every shard to rank 0
is timed separately (`gather`).

Timing: W untimed warm-up steps, then K steps bracketed by barrier + synchronize, CUDA
events on the launching stream, max over ranks. Every step reads inputs larger than
2x the 126 MB L2 (rotating distinct buffers when one batch is smaller). Launches are
replayed through a CUDA graph (the kernel count is unchanged).

The JSON line also carries `roofline` (dominant kernel: algorithmic bytes 2*sizeof(pixel)
per pixel vs the measured HBM copy peak, plus the ALU / issue floors from the committed
ncu capture and the static min/max instruction count of the selection method),
`cpu_baseline` (the C restatement of the reference algorithm, 1 core, bounded sample),
`e2e` (the same metric through the C ABI with pinned host buffers, H2D + D2H inside the
timed region), `gpu_launches` and `clocks`.

`--impl reference` times the reference algorithm's CPU implementation — the oracle port
(oracle/fnr_oracle.c: introsort medians, row-band threads) on every host thread — on the
same config and metric; its input comes from the oracle library (no product library is
loaded). When the unmodified reference package is installed in baseline/_ref, its own
`run_filter` is timed beside it on a bounded sample (`python_reference`).
"""

from __future__ import annotations

import argparse
import ctypes
import json
import math
import os
import statistics
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402

METRIC = "Mpix/s filtered (detect+median)"
L2_BYTES = 126 * 1024 * 1024
FALLBACK_HBM_GBS = 6650.0
SM_COUNT, SM_MHZ = 148, 1965.0
DATA = "synthetic (seeded IR scenes with the BASELINE.json shapes and noise models, DESIGN.md §5)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--method", default="fnr", choices=["fnr", "mf"],
                    help="filter method (run_filter's `method`); the metric is quoted on fnr")
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU-baseline sample budget (seconds of single-core oracle work)")
    ap.add_argument("--ref-seconds", type=float, default=4.0,
                    help="python_reference sample budget per step (reference arm)")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--passes", type=int, default=1,
                    help="filter passes per step (run_filter passes; the CLI default is 2). value counts "
                         "pixel-passes per second")
    ap.add_argument("--multipass", action="store_true",
                    help="passes > 1 as ONE persistent multi-pass launch (irdn_set_multipass; DESIGN.md §9)")
    ap.add_argument("--path", default="filter", choices=["filter", "noise", "sqerr"],
                    help="filter (default, the BASELINE metric) or a widened row (bench_aux.py)")
    return ap.parse_args()


def default_steps(cfg) -> int:
    # aim for a timed region of ~0.4-1 s so clocks can be sampled under load
    return {"c1": 20000, "c2": 20000, "c3": 2000, "c4": 2000, "c5": 600}[cfg.name]


# ---------------------------------------------------------------------------
# Work split and the config block both arms report
# ---------------------------------------------------------------------------
def band_bounds(n: int, parts: int) -> list[int]:
    """The reference's row-band bounds n*i//parts (filters.py:116)."""
    return [n * i // parts for i in range(parts + 1)]


def rank_share(cfg, world: int, rank: int) -> dict:
    """What `rank` filters: a frame range, a row strip (+ halo), or a replica of the workload."""
    if world == 1 or cfg.name == "c1":
        return {"kind": "frames", "f0": 0, "f1": cfg.frames, "replica": world > 1}
    if cfg.frames > 1:
        b = band_bounds(cfg.frames, world)
        return {"kind": "frames", "f0": b[rank], "f1": b[rank + 1], "replica": False}
    b = band_bounds(cfg.height, world)
    r = cfg.k // 2
    y0, y1 = b[rank], b[rank + 1]
    return {"kind": "rows", "y0": y0, "y1": y1, "in0": max(0, y0 - r), "in1": min(cfg.height, y1 + r),
            "replica": False}


def parallelism(cfg, world: int) -> str:
    if world == 1:
        return "1 GPU"
    if cfg.name == "c1":
        return f"replicas x{world} (one 512x512 frame per GPU; SURVEY.md §8e: replicas only)"
    if cfg.frames > 1:
        return f"frame-sharded over {world} GPUs ({cfg.frames} frames split {cfg.frames}/{world})"
    return f"row strips over {world} GPUs ({cfg.height}/{world} rows + {cfg.k // 2}-row halos, global clamp)"


def scaling_kind(cfg, world: int) -> str:
    return "weak" if (cfg.name == "c1" and world > 1) else "strong"


def config_block(cfg, world: int, passes: int, method: str = "fnr") -> dict:
    """Identical in both arms (the driver compares the arms' config)."""
    return {"workload": f"{cfg.name}: {cfg.description}", "frames": cfg.frames, "height": cfg.height,
            "width": cfg.width, "dtype": cfg.dtype, "k": cfg.k, "method": method, "passes": passes,
            "parallelism": parallelism(cfg, world)}


def job_pixels(cfg, world: int) -> int:
    """Pixels of one step summed over all ranks (replicas count once per rank)."""
    return cfg.frames * cfg.height * cfg.width * (world if cfg.name == "c1" else 1)


# ---------------------------------------------------------------------------
# Static selection-method op counts (SURVEY.md §8d anti-gaming guard)
# ---------------------------------------------------------------------------
# Packed min/max instructions (VIMNMX / VIMNMX3 .U16x2, two pixels each) per two output
# pixels, from the kernels' static schedule:
#   dense 3x3 (fnr_k3.cuh, row-first; 160-row tiles: FNR 40 output rows + 2 halo rows per
#     thread, MF 20 + 2): row sort 2 x (rows + 2) / rows, max of lows / min of highs 2, median
#     of the three row middles 3 (sorted shared pair + clamp), final median-of-3 2, FNR: window
#     min / max for the detector 2
#   warp kernel k = 5..11 (fnr_warp.cuh, 64 x 32 tiles, 64 x 48 for k = 11, pixel pairs): detector
#     (K-1)(1 + 2r/rows) horizontal + (K-1) vertical + 1 flag test per pair, plus the median
#     network for two flagged pixels (select_nets.cuh) times the detected fraction.
NET_INSTR_PER_PAIR = {3: 30, 5: 172, 7: 514, 9: None, 11: 1833}
# dense median stage (fnr_dense.cuh, sep_nets.cuh; k = 5 / 7): VIMNMX instructions per output
# pair (tools/netgen/sepgen.py prints them), taken by MF always and by FNR tiles whose
# flagged fraction exceeds DENSE_FRAC (fnr_fast.cuh dense_min_for)
DENSE_INSTR_PER_PAIR = {5: 56.0, 7: 121.5}
# of which emitted as a + b - min (one add, one IMAD: FMA pipe) instead of a second VIMNMX
# (sepgen.py ADDSUB_FRAC = 0.3): the count above stays the method's min / max work
DENSE_ADDSUB_PER_PAIR = {5: 6.5, 7: 15.0}
DENSE_FRAC = {5: 0.20, 7: 0.18}
# FNR tiles predicted dense take the detector from the sorted rows (fnr_dense.cuh FUSED):
# window min / max shared within a group, the noisy test, the signal / changed lanes
FUSED_DET_PER_PAIR = {5: 6.0, 7: 5.5}


def static_ops(cfg, detected_fraction: float, method: str = "fnr") -> dict:
    if cfg.k == 3 and cfg.dtype == "u8":
        # row sort 2 x (rows + 2) / rows per thread (160-row tiles: MF 20 rows, FNR 40), max3 lo,
        # min3 hi, middles 3, final 2, FNR: + min3 lo / max3 hi for the detector
        per_pair = (2 * 22 / 20 + 2 + 3 + 2) if method == "mf" else (2 * 42 / 40 + 2 + 3 + 2 + 2)
        return {"method": ("dense sorted-rows 3x3 median" if method == "mf" else
                           "dense sorted-rows 3x3 median + extremum detector") + " (every pixel)",
                "minmax_instr_per_px": round(per_pair / 2, 3),
                "minmax_lane_ops_per_px": round(per_pair, 3),
                "note": "VIMNMX(3).U16x2 instructions per pixel (each covers 2 pixels); lane ops per pixel"}
    K, r = cfg.k, cfg.k // 2
    tile_rows = 48 if K >= 11 else 32  # fnr_warp.cuh WHK<K>
    det = (K - 1) * (1 + 2 * r / tile_rows) + (K - 1) + 1
    net = NET_INSTR_PER_PAIR.get(K)
    dense = DENSE_INSTR_PER_PAIR.get(K)
    if dense is not None and (method == "mf" or detected_fraction > DENSE_FRAC[K]):
        per_pair = dense + (FUSED_DET_PER_PAIR[K] if method == "fnr" else 0.0)
        return {"method": f"separable {K}x{K} median of every pixel pair from shared sorted rows "
                          f"({dense} instructions per two medians)"
                          + (" + extremum detector fused from the sorted rows" if method == "fnr" else ""),
                "minmax_instr_per_px": round(per_pair / 2, 3), "minmax_lane_ops_per_px": round(per_pair, 3),
                "maxima_as_add_sub_per_px": DENSE_ADDSUB_PER_PAIR[K] / 2,
                "detected_fraction": round(detected_fraction, 4)}
    per_pair = (net or 0) if method == "mf" else det + (net or 0) * detected_fraction  # MF: every pixel, no detector
    return {"method": (f"generated selection network on every pixel pair ({net} instructions per two medians)"
                       if method == "mf" else
                       f"separable {K}x{K} extremum detector on every pixel pair + generated selection "
                       f"network on the flagged pairs ({net} instructions per two medians)"),
            "minmax_instr_per_px": round(per_pair / 2, 3), "minmax_lane_ops_per_px": round(per_pair, 3),
            "detected_fraction": round(detected_fraction, 4)}


def read_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def read_profile(cfg_name: str) -> dict:
    """Per-launch figures of the dominant kernel from the committed ncu capture."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(cfg_name) or {}
    except Exception:
        return {}


class ClockSampler:
    """Samples SM clocks and throttle reasons with NVML while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4,
        "hw_slowdown": 0x8, "sync_boost": 0x10, "sw_thermal_slowdown": 0x20,
        "hw_thermal_slowdown": 0x40, "hw_power_brake_slowdown": 0x80,
        "display_clock_setting": 0x100,
    }

    def __init__(self, index: int):
        self.samples: list[int] = []
        self.reasons: set[str] = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception as e:  # pragma: no cover - no NVML
            self.nvml = None
            self.err = str(e)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nvml.nvmlDeviceGetClockInfo(self.h, self.nvml.NVML_CLOCK_SM))
                mask = self.nvml.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for name, bit in self.REASONS.items():
                    if mask & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.nvml:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()

    def stop(self):
        if self._t:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.nvml:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "note": "NVML unavailable"}
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples), "source": "NVML during the timed region"}


_BACKEND = None


def dist_setup():
    """One rank per GPU (torchrun). NCCL carries the barrier / max-over-ranks timing and the
    separately timed gather; if fewer GPUs than ranks are visible (a code-path check on a
    1-GPU box) ranks share the GPU and the control plane falls back to gloo."""
    global _BACKEND
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        ngpu = torch.cuda.device_count() if torch.cuda.is_available() else 0
        _BACKEND = "nccl" if ngpu >= world else "gloo"
        dist.init_process_group(_BACKEND)
        if ngpu:
            local = local % ngpu
    return world, rank, local


def _max_over_ranks(value: float, dev) -> float:
    import torch
    import torch.distributed as dist

    t = torch.tensor([value], dtype=torch.float64, device=dev if _BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _gather_sum(values: list[int], dev) -> list[int]:
    """Sum small integer vectors on the host: all_gather (no reduction collective), then add."""
    import torch
    import torch.distributed as dist

    t = torch.tensor(values, dtype=torch.int64, device=dev if _BACKEND == "nccl" else "cpu")
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    return [int(x) for x in torch.stack(parts).cpu().sum(0).tolist()]


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference algorithm restated in C; test/baseline only)
# ---------------------------------------------------------------------------
def cpu_sample_run(cfg, frames: np.ndarray, budget_s: float, method: str = "fnr"):
    """One-thread oracle port over a bounded sample; returns (pixels, seconds, description)."""
    from oracle import oracle

    t0 = time.perf_counter()
    px = 0
    if frames.shape[0] == 1 and cfg.height * cfg.width > (4 << 20):
        frame = frames[0]
        y, band = 0, 16
        while time.perf_counter() - t0 < budget_s and y < frame.shape[0]:
            oracle.filter_rows_c(frame, cfg.k, y, min(frame.shape[0], y + band))
            px += min(band, frame.shape[0] - y) * cfg.width
            y += band
        desc = f"{px // cfg.width} rows x {cfg.width} of the {cfg.height}x{cfg.width} frame (row bands)"
    else:
        n = 0
        while time.perf_counter() - t0 < budget_s and n < frames.shape[0]:
            oracle.run_filter_c(frames[n], cfg.k, method, 1, threads=1)
            px += cfg.height * cfg.width
            n += 1
        desc = f"{n} frame(s) of {cfg.height}x{cfg.width} {cfg.dtype}"
    return px, time.perf_counter() - t0, desc


def _pyref_worker(args):
    """One process of the python_reference leg: the UNMODIFIED reference package
    (baseline/_ref) filtering a crop of `rows` output rows with r context rows."""
    ref_path, crop, dtype, k, r_top, rows = args
    sys.path.insert(0, ref_path)
    import irdenoise as ird  # noqa: F401  (the reference, pip-installed into baseline/_ref)
    from irdenoise import image as rimg
    from irdenoise import filters as rfil
    from irdenoise import sorting as rsort

    h, w = crop.shape
    t0 = time.perf_counter()
    if dtype == "u8":
        img = rimg.GrayImage(w, h, bytearray(crop.tobytes()))
        rfil.run_filter(img, rimg.WindowSpec(k), "fnr", 1, threads=1)
    else:
        # u16: the reference's dtype-agnostic per-window API (SURVEY.md §8c u16 oracle)
        class Img:
            pass
        from array import array
        im = Img()
        im.width, im.height, im.pixels = w, h, array("H", crop.tobytes())
        spec = rimg.WindowSpec(k)
        st = rfil.FilterStats()
        sc = rsort.SortCounters()
        for y in range(r_top, r_top + rows):
            for x in range(w):
                win = rimg.extract_window(im, x, y, spec)
                if rfil.classify_pixel(win, rfil.window_extrema(win, st)):
                    rsort.median_of(win.values, sc)
    return rows * w, time.perf_counter() - t0


def python_reference_leg(cfg, frames: np.ndarray, budget_s: float):
    """Time the unmodified reference (baseline/_ref) with one process per host core on a
    bounded sample: each worker filters a crop of the workload's frames (whole frames for
    u8 run_filter, rows + r context rows for the u16 per-window path)."""
    ref_path = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_path, "irdenoise")):
        return {"unavailable": "reference not installed in baseline/_ref (DESIGN.md §3)"}
    import multiprocessing as mp

    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    r = cfg.k // 2
    # per-core rate: ~0.3 Mpix/s at k=3 down to ~0.015 at k=11 (u16); size crops for the budget
    rate = {3: 0.28e6, 5: 0.07e6, 7: 0.08e6, 11: 0.015e6}.get(cfg.k, 0.05e6)
    rows = max(1, min(cfg.height, int(rate * budget_s * 0.6 / cfg.width)))
    jobs = []
    for i in range(cores):
        f = frames[i % frames.shape[0]]
        y0 = (i * 37) % max(1, cfg.height - rows + 1)
        a, b = max(0, y0 - r), min(cfg.height, y0 + rows + r)
        jobs.append((ref_path, np.ascontiguousarray(f[a:b]), cfg.dtype, cfg.k, y0 - a,
                     rows if cfg.dtype != "u8" else b - a))
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        res = pool.map(_pyref_worker, jobs)
    wall = time.perf_counter() - t0
    px = sum(p for p, _ in res)
    per_proc = statistics.median(p / s for p, s in res)
    return {"value": round(px / wall / 1e6, 4), "unit": "Mpix/s", "cores": cores,
            "per_core_value": round(per_proc / 1e6, 4),
            "sample": f"{cores} processes x {rows if cfg.dtype != 'u8' else 'crop of'} rows x {cfg.width} "
                      f"({'run_filter on GrayImage crops' if cfg.dtype == 'u8' else 'per-window API'}), "
                      f"wall {wall:.1f} s incl. process start",
            "source": "unmodified irdenoise 0.1.0 from baseline/_ref (pip install --target)"}


def run_reference_arm(args, cfg, rank: int, world: int):
    if rank != 0:
        return 0
    from oracle import oracle
    from paper_1201_3972_b200.scene import generate

    olib = oracle.lib()  # oracle port + the same seeded scene source; no product library
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    steps = args.steps if args.steps is not None else 5
    if cfg.frames == 1 and cfg.height * cfg.width > (4 << 20):
        frame = generate(cfg, nframes=1, lib=olib)[0]
        rows = 64 * threads
        sample_frames = frame[None, : rows + cfg.k]

        def step():
            ts = []
            per = rows // threads
            for i in range(threads):
                a = i * per
                t = threading.Thread(target=oracle.filter_rows_c, args=(frame, cfg.k, a, a + per))
                t.start()
                ts.append(t)
            for t in ts:
                t.join()
            return rows * cfg.width
        sample = f"{rows} rows x {cfg.width} of the {cfg.height}x{cfg.width} frame per step, {threads} threads"
    else:
        probe = generate(cfg, nframes=1, lib=olib)
        t0 = time.perf_counter()
        oracle.run_filter_c(probe, cfg.k, args.method, 1, threads=threads)
        dt = time.perf_counter() - t0
        nfr = int(max(1, min(cfg.frames, math.ceil(1.0 / max(dt, 1e-4)))))
        frames = generate(cfg, nframes=nfr, lib=olib)
        sample_frames = frames

        def step():
            oracle.run_filter_c(frames, cfg.k, args.method, 1, threads=threads)
            return nfr * cfg.height * cfg.width
        sample = f"{nfr} of {cfg.frames} frame(s) {cfg.height}x{cfg.width} {cfg.dtype} per step, {threads} threads (row bands)"
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    px = 0
    for _ in range(steps):
        px += step()
    dt = time.perf_counter() - t0
    value = px / dt / 1e6
    pyref = python_reference_leg(cfg, sample_frames, args.ref_seconds)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mpix/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(dt / steps * 1e3, 3), "higher_is_better": True, "scaling": scaling_kind(cfg, world),
        "vs_baseline": None, "dtype": cfg.dtype, "data": DATA,
        "config": config_block(cfg, world, 1, args.method),
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpix/s", "cores": threads, "kind": "port",
                         "sample": sample,
                         "note": "oracle/fnr_oracle.c: C restatement of the reference's run_filter "
                                 "(introsort medians, row-band threads); the reference is pure Python"},
        "python_reference": pyref,
        "e2e": {"value": round(value, 4), "unit": "Mpix/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------
def run_b200_arm(args, cfg, rank: int, world: int, local: int):
    import torch

    from paper_1201_3972_b200 import _native
    from paper_1201_3972_b200.scene import render_device

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.load_lib()
    if args.multipass:
        lib.irdn_set_multipass(1)
    steps = args.steps if args.steps is not None else default_steps(cfg)
    warmup = max(3, args.warmup)
    passes = max(1, args.passes)
    share = rank_share(cfg, world, rank)
    bpp = cfg.bytes_per_pixel
    H, W = cfg.height, cfg.width
    # The scene is rendered on the device (irdn_scene_render: the same bytes as the host
    # generator, tests/test_scene_device.py); the pinned host copy feeds the e2e leg and the
    # CPU sample.
    if share["kind"] == "frames":
        B = share["f1"] - share["f0"]
        d0 = render_device(cfg, frame0=share["f0"], nframes=B, device=local)
        out_rows = H
        rank_px = B * H * W
    else:
        if passes > 1:
            raise SystemExit("row strips (c4 at N > 1) are benchmarked with passes = 1")
        B = 1
        full = render_device(cfg, nframes=1, device=local)
        d0 = full[:, share["in0"]:share["in1"]].contiguous()
        del full
        out_rows = share["y1"] - share["y0"]
        rank_px = out_rows * W
    if bpp == 2:
        d0 = d0.view(torch.int16)  # u16 pixels travel as int16 bit patterns
    h_in = torch.empty(d0.shape, dtype=d0.dtype, pin_memory=True)
    h_in.copy_(d0)
    host = h_in.numpy() if bpp == 1 else h_in.numpy().view(np.uint16)
    in_bytes = d0.numel() * bpp
    out_shape = (B, out_rows, W)
    R = max(1, math.ceil(2 * L2_BYTES / (in_bytes + rank_px * bpp)))
    ins = [d0] + [d0.clone() for _ in range(R - 1)]
    outs = [torch.empty(out_shape, dtype=d0.dtype, device=dev) for _ in range(R)]
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    tmp = torch.empty_like(outs[0]) if passes > 1 else None
    stream = torch.cuda.Stream(dev)
    sptr = stream.cuda_stream
    t = "u8" if bpp == 1 else "u16"
    fpass = getattr(lib, f"irdn_filter_pass_{t}")
    M = _native.METHODS[args.method]
    fdev = getattr(lib, f"irdn_run_filter_device_{t}")
    fstrip = getattr(lib, f"irdn_filter_strip_{t}")

    def launch(i: int):
        src, dst = ins[i % R].data_ptr(), outs[i % R].data_ptr()
        if share["kind"] == "rows":
            rc = fstrip(src, share["in0"], share["in1"] - share["in0"], dst, share["y0"], share["y1"], H, W, W, W,
                        cfg.k, M, counts.data_ptr(), sptr)
        elif passes == 1:
            rc = fpass(src, dst, B, H, W, W, W, cfg.k, M, counts.data_ptr(), sptr)
        else:  # run_filter over device buffers: passes back-to-back launches through tmp
            rc = fdev(src, dst, tmp.data_ptr(), B, H, W, cfg.k, M, passes, counts.data_ptr(), sptr)
        if rc != 0:
            _native.check(rc)

    with torch.cuda.stream(stream):
        for i in range(warmup):
            launch(i)
    torch.cuda.synchronize(dev)
    lib.irdn_reset_launch_count()
    with torch.cuda.stream(stream):
        launch(0)
    torch.cuda.synchronize(dev)
    per_step = int(lib.irdn_launch_count())

    graph = None
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=stream):
                for i in range(R):
                    launch(i)
            torch.cuda.synchronize(dev)
            graph.replay()
            torch.cuda.synchronize(dev)
        except Exception as e:  # capture failure: eager launches
            sys.stderr.write(f"graph capture failed ({e}); timing eager launches\n")
            graph = None

    counts.zero_()
    torch.cuda.synchronize(dev)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    sampler = ClockSampler(local)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    lib.irdn_reset_launch_count()
    sampler.start()
    torch.cuda.synchronize(dev)
    with torch.cuda.stream(stream):
        ev0.record(stream)
        if graph is not None:
            for _ in range(steps // R):
                graph.replay()
            for i in range(steps % R):
                launch(i)
        else:
            for i in range(steps):
                launch(i)
        ev1.record(stream)
    torch.cuda.synchronize(dev)
    sampler.stop()
    eager_launches = int(lib.irdn_launch_count())
    gpu_launches = ((steps // R) * R + (steps % R)) * per_step if graph is not None else eager_launches
    rank_ms = ev0.elapsed_time(ev1)
    elapsed_ms = rank_ms
    det_rank = int(counts[0].item())
    det_total = det_rank
    if world > 1:
        elapsed_ms = _max_over_ranks(rank_ms, dev)
        det_total = _gather_sum([det_rank], dev)[0]
    ms_per_step = elapsed_ms / steps
    value = job_pixels(cfg, world) * passes * steps / (elapsed_ms * 1e-3) / 1e6

    # gather: every rank's output shard to rank 0 (outputs otherwise stay sharded), timed alone
    gather = None
    if world > 1:
        gather = time_gather(outs[0], dev, rank, world, share, cfg)
        if passes == 1:
            gather["fused"] = time_fused_gather(ins[0], dev, rank, world, share, cfg, lib, _native, M, counts, sptr)

    # the dominant kernel: this rank's per-launch average over the timed region; isolated
    # per-launch events (which defeat the programmatic-dependent-launch overlap) beside it
    nper = min(steps, 200)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nper)]
    with torch.cuda.stream(stream):
        for i in range(nper):
            evs[i][0].record(stream)
            launch(i)
            evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    per = [a.elapsed_time(b) / passes for a, b in evs]
    kernel_ms = rank_ms / (steps * passes)

    peak, peak_src = read_peaks()
    alg_bytes = rank_px * 2 * bpp
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    prof = read_profile(cfg.name)
    traffic = prof.get("dram_bytes_per_launch")
    if traffic is not None and prof.get("pixels_per_launch"):
        traffic = traffic * rank_px / prof["pixels_per_launch"]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": round(traffic) if traffic else None,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes, "bytes_per_pixel": 2 * bpp,
                "pixels_per_launch": rank_px,
                "kernel_ms": round(kernel_ms, 5),
                "kernel_ms_source": "CUDA events on the launching stream over the timed region / filter launches",
                "kernel_ms_isolated": round(statistics.mean(per), 5),
                "kernel_ms_isolated_min": round(min(per), 5),
                "static_ops": static_ops(cfg, det_rank / max(1, rank_px * steps * passes), args.method)}
    # the method's own min/max work against the ALU pipe (the anti-gaming guard is
    # the STATIC count of the selection method, not the executed instruction count)
    so = roofline["static_ops"]
    alu_lanes = 64 * SM_COUNT * SM_MHZ * 1e6  # thread-instructions / s on the ALU pipe
    so["alu_floor_us"] = round(so["minmax_instr_per_px"] * rank_px / alu_lanes * 1e6, 2)
    so["frac"] = round(so["minmax_instr_per_px"] * rank_px / (kernel_ms * 1e-3) / alu_lanes, 4)
    if prof.get("instr_per_px") and args.method == "fnr" and passes == 1:  # the captures are single FNR passes
        # SM-side floors from the committed capture (instructions / ALU-pipe instructions per pixel)
        ipp, app = prof["instr_per_px"], prof.get("alu_instr_per_px")
        issue_peak = 128 * SM_COUNT * SM_MHZ * 1e6
        alu_peak = 64 * SM_COUNT * SM_MHZ * 1e6
        roofline["issue"] = {"instr_per_px": round(ipp, 2), "frac": round(ipp * rank_px / (kernel_ms * 1e-3) / issue_peak, 4),
                             "floor_us": round(ipp * rank_px / issue_peak * 1e6, 2),
                             "peak": "4 warp-instructions/clk/SM x 148 SMs x 1965 MHz"}
        if app:
            roofline["alu"] = {"alu_instr_per_px": round(app, 2),
                               "frac": round(app * rank_px / (kernel_ms * 1e-3) / alu_peak, 4),
                               "floor_us": round(app * rank_px / alu_peak * 1e6, 2),
                               "peak": "2 warp-instructions/clk/SM (VIMNMX/PRMT/IADD3/LOP3, "
                                       "profiles/pipe_probe_r02.txt) x 148 x 1965 MHz"}
        roofline["profile"] = prof.get("source")

    e2e = run_e2e(args, cfg, lib, _native, h_in, outs[0], share, steps, dev, world, passes, local)
    e2e_det = e2e.pop("_detected")
    if e2e_det is not None and e2e_det * steps != det_rank:
        raise AssertionError("counter mismatch between the device-resident and the host-buffer path")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle

        oracle.lib()
        px, secs, desc = cpu_sample_run(cfg, host, args.cpu_seconds, args.method)
        cpu = {"value": round(px / secs / 1e6, 4), "unit": "Mpix/s", "cores": 1, "kind": "port",
               "sample": desc + f" ({secs:.1f} s)",
               "note": "oracle/fnr_oracle.c (reference algorithm restated in C: clamp gather, "
                       "min/max detector, introsort median), single thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mpix/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": scaling_kind(cfg, world), "vs_baseline": None,
            "dtype": cfg.dtype, "data": DATA,
            "config": config_block(cfg, world, passes, args.method),
            "run": {"pixels_per_step": job_pixels(cfg, world), "rank0_share": share,
                    "detected_per_step": det_total // steps,
                    "l2": f"rotating {R} distinct in/out buffers ({(in_bytes + rank_px * bpp) * R / 1e6:.0f} MB > 2x L2)"
                          if R > 1 else f"in+out {(in_bytes + rank_px * bpp) / 1e6:.0f} MB per step > 2x L2",
                    "launch": "CUDA graph of R launches" if graph is not None else "eager",
                    **({"multipass_launch": True} if args.multipass and passes > 1 else {}),
                    "collective_backend": _BACKEND},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches * world, "clocks": sampler.summary(),
        }
        if gather is not None:
            line["gather"] = gather
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()
    return 0


def time_gather(out, dev, rank: int, world: int, share: dict, cfg):
    """One gather of every rank's output shard to rank 0 (P2P over NVLink through NCCL on a
    multi-GPU node; through the host with the gloo fallback), timed on its own."""
    import torch
    import torch.distributed as dist

    flat = out.reshape(-1).view(torch.uint8)  # bytes: gloo has no 16-bit integer collectives
    n = torch.tensor([flat.numel()], dtype=torch.int64, device=dev if _BACKEND == "nccl" else "cpu")
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    send = flat if _BACKEND == "nccl" else flat.cpu()
    if send.numel() < mx:
        send = torch.cat([send, send.new_zeros(mx - send.numel())])
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    for _ in range(2):  # warm-up (connection setup)
        dist.gather(send, bufs, dst=0)
    torch.cuda.synchronize(dev)
    dist.barrier()
    t0 = time.perf_counter()
    dist.gather(send, bufs, dst=0)
    torch.cuda.synchronize(dev)
    secs = _max_over_ranks(time.perf_counter() - t0, dev)
    bytes_in = sum(sizes)
    return {"ms": round(secs * 1e3, 3), "bytes": bytes_in, "backend": _BACKEND,
            "note": "outputs stay sharded during the filter; this is one gather to rank 0, "
                    "not included in value"}


def time_fused_gather(src, dev, rank: int, world: int, share: dict, cfg, lib, _native, M, counts, sptr):
    """The gather fused into the filter: rank 0's full output is mapped into every rank
    (CUDA IPC, irdn_ipc_*) and each rank's filter launch stores its shard straight into it
    (NVLink peer stores tile by tile). Timed from a common barrier to the last rank's
    completion (host clock around a synchronised launch, max over ranks); compare with
    value's filter-only time plus `gather.ms`."""
    import ctypes

    import torch
    import torch.distributed as dist

    H, W, bpp = cfg.height, cfg.width, cfg.bytes_per_pixel
    full = torch.empty((cfg.frames if cfg.frames > 1 else 1, H, W), dtype=src.dtype, device=dev) if rank == 0 else None
    msg = [None]
    if rank == 0:
        handle, off = ctypes.create_string_buffer(64), ctypes.c_uint64(0)
        if lib.irdn_ipc_export(full.data_ptr(), handle, ctypes.byref(off)) == 0:
            msg = [(handle.raw, int(off.value))]
    dist.broadcast_object_list(msg, src=0)
    base, why = None, None
    if msg[0] is None:
        why = "rank 0 could not export its output buffer"
    else:
        raw, off = msg[0]
        if rank == 0:
            base = full.data_ptr()
        else:
            ptr = ctypes.c_void_p()
            if lib.irdn_ipc_open(ctypes.create_string_buffer(raw, 64), off, ctypes.byref(ptr)) == 0:
                base = ptr.value
            else:
                why = _native.load_lib().irdn_last_error().decode()
    oks = [None] * world
    dist.all_gather_object(oks, base is not None)  # every rank agrees before any peer store
    if not all(oks):
        if base is not None and rank != 0:
            lib.irdn_ipc_close(ctypes.c_void_p(base), off)
        return {"unavailable": why or "a peer could not map rank 0's output (no CUDA IPC / P2P)"}
    t = "u8" if bpp == 1 else "u16"
    try:
        def launch():
            if share["kind"] == "rows":
                fn = getattr(lib, f"irdn_filter_strip_{t}")
                dst = base + share["y0"] * W * bpp
                _native.check(fn(src.data_ptr(), share["in0"], share["in1"] - share["in0"], dst, share["y0"],
                                 share["y1"], H, W, W, W, cfg.k, M, counts.data_ptr(), sptr))
            else:
                nfr = share["f1"] - share["f0"]
                if share.get("replica"):
                    dst = base  # replicas (c1): every rank writes the same frame
                else:
                    dst = base + share["f0"] * H * W * bpp
                fn = getattr(lib, f"irdn_filter_pass_{t}")
                _native.check(fn(src.data_ptr(), dst, nfr, H, W, W, W, cfg.k, M, counts.data_ptr(), sptr))
        for _ in range(2):
            launch()
        torch.cuda.synchronize(dev)
        dist.barrier()
        t0 = time.perf_counter()
        launch()
        torch.cuda.synchronize(dev)
        secs = _max_over_ranks(time.perf_counter() - t0, dev)
        dist.barrier()
    finally:
        if rank != 0:
            lib.irdn_ipc_close(ctypes.c_void_p(base), off)
    return {"ms": round(secs * 1e3, 3),
            "note": "filter launch with every rank storing its shard into rank 0's output "
                    "(CUDA IPC mapping, NVLink peer stores); host clock, max over ranks"}


def run_e2e(args, cfg, lib, _native, h_in, d_out_ref, share, steps, dev, world, passes, local):
    """e2e: the same metric through the C ABI with pinned host buffers, H2D + D2H timed."""
    import torch

    bpp = cfg.bytes_per_pixel
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(steps, 10 if h_in.numel() * bpp > (256 << 20) else 40))
    t = "u8" if bpp == 1 else "u16"
    H, W = cfg.height, cfg.width
    M = _native.METHODS[args.method]
    if share["kind"] == "rows":
        # a row strip: H2D of the strip (+ halo rows), irdn_filter_strip_*, D2H of the owned rows
        fstrip = getattr(lib, f"irdn_filter_strip_{t}")
        rows = share["y1"] - share["y0"]
        h_out = torch.empty((1, rows, W), dtype=h_in.dtype).pin_memory()
        d_in = torch.empty_like(h_in, device=dev)
        d_out = torch.empty((1, rows, W), dtype=h_in.dtype, device=dev)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        s = torch.cuda.current_stream(dev)

        def call():
            d_in.copy_(h_in, non_blocking=True)
            _native.check(fstrip(d_in.data_ptr(), share["in0"], share["in1"] - share["in0"], d_out.data_ptr(),
                                 share["y0"], share["y1"], H, W, W, W, cfg.k, M, counts.data_ptr(), s.cuda_stream))
            h_out.copy_(d_out, non_blocking=True)
            s.synchronize()
        call()
        if world > 1:
            import torch.distributed as dist

            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            call()
        secs = time.perf_counter() - t0
        if world > 1:
            secs = _max_over_ranks(secs, dev)
        if not torch.equal(h_out.to(dev), d_out_ref):
            raise AssertionError("e2e strip output differs from the device-resident output")
        return {"value": round(job_pixels(cfg, world) * e2e_steps / secs / 1e6, 3), "unit": "Mpix/s",
                "h2d_bytes_per_step": h_in.numel() * bpp, "d2h_bytes_per_step": rows * W * bpp,
                "steps": e2e_steps, "_detected": None,
                "api": f"irdn_filter_strip_{t} (C ABI) between pinned host buffers; host wall clock"}

    B = share["f1"] - share["f0"]
    h_out = torch.empty_like(h_in).pin_memory()
    st = _native.IrdnStats()
    hfn = getattr(lib, f"irdn_run_filter_{t}")
    for _ in range(2):
        _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, M, passes, local, ctypes.byref(st)))

    def e2e_run(mode: str):
        prev = _native.set_host_return(mode)
        try:
            _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, M, passes, local,
                              ctypes.byref(st)))
            if world > 1:
                import torch.distributed as dist

                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, M, passes, local,
                                  ctypes.byref(st)))
            secs = time.perf_counter() - t0
            if world > 1:
                secs = _max_over_ranks(secs, dev)
            h2d, d2h = _native.last_transfer()
        finally:
            _native.set_host_return(prev)
        if passes == 1 and not torch.equal(h_out.to(dev), d_out_ref):
            raise AssertionError(f"e2e output ({mode} return) differs from the device-resident output")
        return job_pixels(cfg, world) * passes * e2e_steps / secs / 1e6, h2d, d2h

    full_v, _, full_d2h = e2e_run("full")
    e2e_v, h2d, d2h = e2e_run("auto")
    batch_bytes = h_in.numel() * bpp
    return {"value": round(e2e_v, 3), "unit": "Mpix/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
            "api": f"irdn_run_filter_{t} (C ABI, include/irdn.h) on pinned host buffers; "
                   "host wall clock, call is synchronous",
            "result_return": "sparse (changed pixels only, rebuilt on the host from its input; DESIGN.md §7.1)"
                             if d2h < batch_bytes else "full D2H copy (auto mode: 8-bit frames, or < 6 host "
                                                       "threads per GPU process; DESIGN.md §7.1)",
            "full_copy": {"value": round(full_v, 3), "d2h_bytes_per_step": full_d2h},
            "_detected": int(st.detected)}


def main():
    args = parse()
    if args.path != "filter":
        import bench_aux

        return {"noise": bench_aux.run_noise, "sqerr": bench_aux.run_sqerr}[args.path](args, sys.modules[__name__])
    from paper_1201_3972_b200.scene import CONFIGS

    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup()
    if args.impl == "reference":
        rc = run_reference_arm(args, cfg, rank, world)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return rc
    return run_b200_arm(args, cfg, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
