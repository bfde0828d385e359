"""Measurements of the widened rows beside the filter: `bench.py --path noise|sqerr`.

    python bench.py --path noise  [--steps K] [--warmup W]   # inject_impulse, Mpix/s
    python bench.py --path sqerr  [--steps K] [--warmup W]   # exact squared-error sum (MSE/PSNR), Mpix/s

Same JSON-line shape and timing rules as the filter bench (bench.py): W >= 3 warm-up
steps, K timed steps on the launching stream with CUDA events, inputs resident in HBM
and larger than 2x L2 per step, NVML clocks during the timed region; `e2e` through the
public API with host buffers (H2D + D2H in the timed region); `cpu_baseline` = the C
oracle restating the reference (1 thread, bounded sample). One GPU (replicas only).

Workloads (seeded synthetic):
  noise  8192 x 8192 u8 image (67 Mpx), NoiseSpec(density 0.2, salt 0.5, seed 42) — the
         reference CLI's add-noise defaults (cli.py:206-212) on a large frame.
  sqerr  8192 x 8192 u16 pair (c4's frame shape), the numerator of metrics.mse.
"""

from __future__ import annotations

import ctypes
import json
import time

import numpy as np


def _timed(stream, steps, launch):
    import torch

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        ev0.record(stream)
        for i in range(steps):
            launch(i)
        ev1.record(stream)
    torch.cuda.synchronize()
    return ev0.elapsed_time(ev1)


def run_noise(args, bench):
    import torch

    from oracle import oracle
    from paper_1201_3972_b200 import _native
    from paper_1201_3972_b200.noise import NoiseSpec, inject_impulse

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = _native.load_lib()
    H = W = 8192
    n = H * W
    spec = NoiseSpec(0.2, 0.5, 42)
    rng = np.random.default_rng(1)
    host = rng.integers(0, 256, n, dtype=np.uint8)
    src = torch.from_numpy(host).to(dev)
    outs = [torch.empty_like(src) for _ in range(2)]
    flags = [torch.empty_like(src) for _ in range(2)]
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(dev)
    steps = args.steps if args.steps is not None else 200
    warmup = max(3, args.warmup)

    def launch(i):
        _native.check(lib.irdn_inject_impulse_u8(src.data_ptr(), outs[i % 2].data_ptr(), flags[i % 2].data_ptr(),
                                                 n, spec.seed, spec.density, spec.salt_fraction,
                                                 cnt.data_ptr(), stream.cuda_stream))

    _timed(stream, warmup, launch)
    cnt.zero_()
    sampler = bench.ClockSampler(0)
    lib.irdn_reset_launch_count()
    sampler.start()
    ms = _timed(stream, steps, launch)
    sampler.stop()
    launches = int(lib.irdn_launch_count())
    corrupted = int(cnt.item()) // steps
    # parity of the measured output against the oracle (whole image)
    want, wflags, wcnt = oracle.inject_impulse_c(host, spec.seed, spec.density, spec.salt_fraction)
    if not (np.array_equal(outs[(steps - 1) % 2].cpu().numpy(), want) and corrupted == wcnt):
        raise AssertionError("inject_impulse output differs from the oracle")
    kernel_ms = ms / steps
    alg = 3 * n  # read the image, write noisy image + mask flags
    peak, peak_src = bench.read_peaks()
    achieved = alg / (kernel_ms * 1e-3) / 1e9
    # e2e: the public API on a GrayImage-sized host buffer (numpy in, numpy out)
    e2e_steps = 5
    inject_impulse(host, spec)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        inject_impulse(host, spec)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    # CPU baseline: the oracle's sequential SplitMix64 walk (the reference algorithm) on a sample
    sample = host[: 16 << 20]
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < min(args.cpu_seconds, 10.0) or reps == 0:
        oracle.inject_impulse_c(sample, spec.seed, spec.density, spec.salt_fraction)
        reps += 1
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": "Mpix/s noised (inject_impulse)", "value": round(n / (kernel_ms * 1e-3) / 1e6, 3),
        "unit": "Mpix/s", "n_gpus": 1, "steps": steps, "warmup": warmup, "ms_per_step": round(kernel_ms, 5),
        "higher_is_better": True, "scaling": "replicas", "vs_baseline": None, "dtype": "u8/u64",
        "data": "synthetic (seeded uniform u8 image)",
        "config": {"workload": "noise: one 8192x8192 u8 image, NoiseSpec(0.2, 0.5, 42) (cli.py add-noise defaults)",
                   "corrupted_per_step": corrupted,
                   "l2": "in 67 MB + out 67 MB + flags 67 MB + bit words 34 MB per step > 2x L2 over 2 steps"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg, "bytes_per_pixel": 3, "kernel_ms": round(kernel_ms, 5),
                     "note": "3 kernels per call (draws, chunk scan, emit); the draws kernel is 64-bit-multiply "
                             "bound: 2 SplitMix64 draws per pixel (2n positions) ~ 60 integer ops/px"},
        "cpu_baseline": {"value": round(reps * sample.size / cpu_s / 1e6, 3), "unit": "Mpix/s", "cores": 1,
                         "kind": "port", "sample": f"{reps} x {sample.size} px ({cpu_s:.1f} s)",
                         "note": "oracle_inject_impulse (noise.py:89-106 restated in C, sequential)"},
        "e2e": {"value": round(n / e2e_s / 1e6, 3), "unit": "Mpix/s", "h2d_bytes_per_step": n,
                "d2h_bytes_per_step": 2 * n, "steps": e2e_steps,
                "api": "paper_1201_3972_b200.inject_impulse(numpy u8) -> (noisy, flags); host wall clock"},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_sqerr(args, bench):
    import torch

    from oracle import oracle
    from paper_1201_3972_b200 import _native, metrics

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    lib = _native.load_lib()
    H = W = 8192
    n = H * W
    rng = np.random.default_rng(2)
    ha = rng.integers(0, 16384, n, dtype=np.uint16)
    hb = rng.integers(0, 16384, n, dtype=np.uint16)
    pairs = []
    for r in range(2):  # 2 pairs x 268 MB > 2x L2
        a = torch.from_numpy(ha.view(np.int16)).to(dev).view(torch.uint16)
        b = torch.from_numpy(hb.view(np.int16)).to(dev).view(torch.uint16)
        pairs.append((a, b))
    acc = torch.zeros(1, dtype=torch.int64, device=dev)
    stream = torch.cuda.Stream(dev)
    steps = args.steps if args.steps is not None else 500
    warmup = max(3, args.warmup)

    def launch(i):
        a, b = pairs[i % 2]
        _native.check(lib.irdn_sq_err_sum_u16(a.data_ptr(), b.data_ptr(), n, acc.data_ptr(), stream.cuda_stream))

    _timed(stream, warmup, launch)
    acc.zero_()
    sampler = bench.ClockSampler(0)
    lib.irdn_reset_launch_count()
    sampler.start()
    ms = _timed(stream, steps, launch)
    sampler.stop()
    launches = int(lib.irdn_launch_count())
    want = oracle.sq_err_sum_c(ha, hb)
    if (int(acc.item()) & 0xFFFFFFFFFFFFFFFF) != (want * steps) & 0xFFFFFFFFFFFFFFFF:
        raise AssertionError("sq_err_sum differs from the oracle")
    kernel_ms = ms / steps
    alg = 4 * n
    peak, peak_src = bench.read_peaks()
    achieved = alg / (kernel_ms * 1e-3) / 1e9
    e2e_steps = 5
    metrics.mse(ha, hb)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        metrics.mse(ha, hb)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    t0 = time.perf_counter()
    reps = 0
    while time.perf_counter() - t0 < min(args.cpu_seconds, 5.0) or reps == 0:
        oracle.sq_err_sum_c(ha, hb)
        reps += 1
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": "Mpix/s compared (exact squared-error sum for MSE/PSNR)",
        "value": round(n / (kernel_ms * 1e-3) / 1e6, 3), "unit": "Mpix/s", "n_gpus": 1, "steps": steps,
        "warmup": warmup, "ms_per_step": round(kernel_ms, 5), "higher_is_better": True, "scaling": "replicas",
        "vs_baseline": None, "dtype": "u16/u64", "data": "synthetic (seeded uniform 14-bit u16 pair)",
        "config": {"workload": "sqerr: one 8192x8192 u16 image pair (metrics.mse numerator)",
                   "l2": "2 rotating pairs x 268 MB > 2x L2"},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes_per_launch": alg, "bytes_per_pixel": 4, "kernel_ms": round(kernel_ms, 5)},
        "cpu_baseline": {"value": round(reps * n / cpu_s / 1e6, 3), "unit": "Mpix/s", "cores": 1, "kind": "port",
                         "sample": f"{reps} x {n} px ({cpu_s:.1f} s)",
                         "note": "oracle_sq_err_sum (metrics.py:29-32 restated in C)"},
        "e2e": {"value": round(n / e2e_s / 1e6, 3), "unit": "Mpix/s", "h2d_bytes_per_step": 4 * n,
                "d2h_bytes_per_step": 8, "steps": e2e_steps,
                "api": "paper_1201_3972_b200.mse(numpy u16, numpy u16); host wall clock"},
        "gpu_launches": launches, "clocks": sampler.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0
