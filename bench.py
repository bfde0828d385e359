#!/usr/bin/env python
"""FNR filter benchmark: Mpix/s filtered (detect + median) on B200, BASELINE.json metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

One "step" is one filter pass (method "fnr", passes=1 — the run_filter default,
filters.py:83) over one batch of the workload. The default workload is
BASELINE.json configs[1] (c2: 64 x 640x512 uint16 14-bit frames, 5x5 window);
`--config c1..c5` selects another BASELINE config. For N > 1 (torchrun, one
rank per GPU) every rank filters its own batch of further frames of the same
seeded stream (frame sharding, no data-path collective: scaling "weak").

Timing: W untimed warm-up steps, then K steps bracketed by barrier +
synchronize, CUDA events on the launching stream, max over ranks. Steps
rotate over R distinct input/output batches whose total size exceeds 2x the
126 MB L2, so every step reads its input from HBM. Launches are replayed
through a CUDA graph of R launches (the kernel count is unchanged).

The JSON line also carries: `roofline` (dominant kernel, algorithmic bytes
2*sizeof(pixel) per pixel vs the measured HBM copy peak), `cpu_baseline`
(the C restatement of the reference algorithm, 1 core, bounded sample), `e2e`
(the same metric through the C-ABI host entry irdn_run_filter_* with pinned
host buffers, H2D + D2H inside the timed region), `gpu_launches`, `clocks`.

`--impl reference` times the reference algorithm's CPU implementation — the
oracle port (oracle/fnr_oracle.c: introsort medians, row-band threads), with
every host thread — on the same config and metric. The reference itself is
pure Python (irdenoise) and cannot be compiled.
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="CPU-baseline sample budget (seconds of single-core oracle work)")
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
    # aim for a timed region of ~0.5-1 s so clocks can be sampled under load
    return {"c1": 20000, "c2": 20000, "c3": 2000, "c4": 1000, "c5": 500}[cfg.name]


def workload_desc(cfg) -> str:
    return f"{cfg.name}: {cfg.description}"


def read_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def read_profile_traffic(cfg_name: str):
    """dram bytes per launch of the dominant kernel from a committed ncu --set full capture."""
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(cfg_name) or {}
        return e.get("dram_bytes_per_launch"), e
    except Exception:
        return None, {}


def read_alu_floor(cfg_name: str):
    """ALU-pipe lane-ops per pixel of the dominant kernel (tools/prof/alu_floor.py output)."""
    import glob

    paths = sorted(glob.glob(os.path.join(REPO, "profiles", "alu_floor_*.json")))
    for path in reversed(paths):  # newest capture tag first
        try:
            for row in json.load(open(path)):
                if row["config"] == cfg_name:
                    return dict(row, source=os.path.relpath(path, REPO) +
                                " (ALU opcodes x 32 lanes from the ncu SASS mix; 64 lanes/clk/SM measured)")
        except Exception:
            continue
    return None


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


def dist_setup(n_gpus: int):
    """One rank per GPU (torchrun). NCCL carries the barrier / max-over-ranks timing; if
    fewer GPUs than ranks are visible (a code-path check on a 1-GPU box) ranks share GPUs
    and the control plane falls back to gloo. No data-path collective either way."""
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


# ---------------------------------------------------------------------------
# CPU legs (oracle = the reference algorithm restated in C; test/baseline only)
# ---------------------------------------------------------------------------
def cpu_sample_run(cfg, frames: np.ndarray, threads: int, budget_s: float, full_frame=None):
    """Run the oracle port over a bounded sample; returns (pixels, seconds, description)."""
    from oracle import oracle

    t0 = time.perf_counter()
    px = 0
    if cfg.frames == 1 and cfg.height * cfg.width > (4 << 20):
        # one huge frame (c4): row bands of the full frame, clamped against the frame
        frame = full_frame if full_frame is not None else frames[0]
        band = 16
        y = 0
        bands = 0
        while time.perf_counter() - t0 < budget_s and y < cfg.height:
            oracle.filter_rows_c(frame, cfg.k, y, min(cfg.height, y + band)) if threads == 1 else \
                _threaded_rows(frame, cfg.k, y, min(cfg.height, y + band * threads), threads)
            rows = band if threads == 1 else band * threads
            px += min(rows, cfg.height - y) * cfg.width
            y += rows
            bands += 1
        desc = f"{px // cfg.width} rows x {cfg.width} of the {cfg.height}x{cfg.width} frame (row bands)"
    else:
        n = 0
        while time.perf_counter() - t0 < budget_s and n < frames.shape[0]:
            oracle.run_filter_c(frames[n], cfg.k, "fnr", 1, threads=threads)
            px += cfg.height * cfg.width
            n += 1
        desc = f"{n} frame(s) of {cfg.height}x{cfg.width} {cfg.dtype}"
    return px, time.perf_counter() - t0, desc


def _threaded_rows(frame, k, y0, y1, threads):
    from oracle import oracle

    # oracle_run_filter splits a frame into row bands itself; for a row range use bands per thread
    ts = []
    step = max(1, (y1 - y0 + threads - 1) // threads)
    for a in range(y0, y1, step):
        t = threading.Thread(target=oracle.filter_rows_c, args=(frame, k, a, min(y1, a + step)))
        t.start()
        ts.append(t)
    for t in ts:
        t.join()


def run_reference_arm(args, cfg, rank: int, world: int):
    if rank != 0:
        return 0
    from oracle import oracle
    from paper_1201_3972_b200.scene import generate

    oracle.lib()
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    steps = args.steps if args.steps is not None else 5
    # sample: whole frames for batch configs, row bands of the frame for c4
    if cfg.frames == 1 and cfg.height * cfg.width > (4 << 20):
        frame = generate(cfg, nframes=1)[0]
        rows = 64 * threads

        def step():
            from oracle import oracle as o

            ts = []
            per = rows // threads
            for i in range(threads):
                a = i * per
                t = threading.Thread(target=o.filter_rows_c, args=(frame, cfg.k, a, a + per))
                t.start()
                ts.append(t)
            for t in ts:
                t.join()
            return rows * cfg.width
        sample = f"{rows} rows x {cfg.width} of the {cfg.height}x{cfg.width} frame per step, {threads} threads"
    else:
        nfr = 1
        probe = generate(cfg, nframes=1)
        t0 = time.perf_counter()
        oracle.run_filter_c(probe, cfg.k, "fnr", 1, threads=threads)
        dt = time.perf_counter() - t0
        nfr = int(max(1, min(cfg.frames, math.ceil(1.0 / max(dt, 1e-4)))))
        frames = generate(cfg, nframes=nfr)

        def step():
            oracle.run_filter_c(frames, cfg.k, "fnr", 1, threads=threads)
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
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "Mpix/s",
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": round(dt / steps * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded IR scenes, DESIGN.md §5)",
        "config": {"workload": workload_desc(cfg), "method": "fnr", "passes": 1, "k": cfg.k},
        "cpu_baseline": {"value": round(value, 4), "unit": "Mpix/s", "cores": threads, "kind": "port",
                         "sample": sample,
                         "note": "oracle/fnr_oracle.c: C restatement of the reference's run_filter "
                                 "(introsort medians, row-band threads); the reference is pure Python"},
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
    from paper_1201_3972_b200.scene import generate

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    lib = _native.load_lib()
    if args.multipass:
        lib.irdn_set_multipass(1)
    steps = args.steps if args.steps is not None else default_steps(cfg)
    warmup = max(3, args.warmup)
    bpp = cfg.bytes_per_pixel
    B, H, W = cfg.frames, cfg.height, cfg.width
    batch_px = B * H * W
    batch_bytes = batch_px * bpp

    # this rank's batch: frames [rank*B, (rank+1)*B) of the seeded stream (c1/c4: replicas)
    frame0 = rank * B if B > 1 else 0
    host = generate(cfg, frame0=frame0, nframes=B)
    h_in = torch.from_numpy(host).pin_memory() if bpp == 1 else \
        torch.from_numpy(host.view(np.int16)).pin_memory()
    d0 = h_in.to(dev, non_blocking=False)  # u16 pixels travel as int16 bit patterns
    R = max(1, math.ceil(2 * L2_BYTES / (2 * batch_bytes)))
    ins = [d0] + [d0.clone() for _ in range(R - 1)]
    outs = [torch.empty_like(d0) for _ in range(R)]
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    fn = lib.irdn_filter_pass_u8 if bpp == 1 else lib.irdn_filter_pass_u16
    dfn = lib.irdn_run_filter_device_u8 if bpp == 1 else lib.irdn_run_filter_device_u16
    passes = max(1, args.passes)
    tmp = torch.empty_like(d0) if passes > 1 else None
    stream = torch.cuda.Stream(dev)
    sptr = stream.cuda_stream

    def launch(i: int):
        if passes == 1:
            rc = fn(ins[i % R].data_ptr(), outs[i % R].data_ptr(), B, H, W, W, W, cfg.k, 0,
                    counts.data_ptr(), sptr)
        else:  # run_filter over device buffers: all passes in one multi-pass launch (via tmp)
            rc = dfn(ins[i % R].data_ptr(), outs[i % R].data_ptr(), tmp.data_ptr(), B, H, W, cfg.k, 0, passes,
                     counts.data_ptr(), sptr)
        if rc != 0:
            _native.check(rc)

    with torch.cuda.stream(stream):
        for i in range(warmup):
            launch(i)
    torch.cuda.synchronize(dev)
    # kernel launches per step (1 for passes > 1 too: all passes run in one multi-pass launch)
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
    elapsed_ms = ev0.elapsed_time(ev1)
    if world > 1:
        import torch.distributed as dist

        elapsed_ms = _max_over_ranks(elapsed_ms, dev)
        dist.barrier()
    det = int(counts[0].item())
    ms_per_step = elapsed_ms / steps
    value = world * batch_px * passes * steps / (elapsed_ms * 1e-3) / 1e6

    # dominant-kernel duration: per-launch CUDA events on the launching stream (separate pass)
    per = []
    nper = min(steps, 200)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(nper)]
    with torch.cuda.stream(stream):
        for i in range(nper):
            evs[i][0].record(stream)
            launch(i)
            evs[i][1].record(stream)
    torch.cuda.synchronize(dev)
    per = [a.elapsed_time(b) / passes for a, b in evs]  # per filter launch, isolated by events
    # the dominant kernel's average launch duration over the timed region: the region
    # holds exactly steps x passes filter launches back to back (programmatic dependent
    # launch overlaps each launch's ramp with the previous one's tail); the isolated
    # per-launch figure (events around every launch defeat that overlap) is kept beside it
    kernel_ms = elapsed_ms / (steps * passes)

    peak, peak_src = read_peaks()
    alg_bytes = batch_px * 2 * bpp
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    traffic, prof = read_profile_traffic(cfg.name)
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "peak_source": peak_src,
                "algorithmic_bytes_per_launch": alg_bytes,
                "bytes_per_pixel": 2 * bpp, "pixels_per_launch": batch_px,
                "kernel_ms": round(kernel_ms, 5),
                "kernel_ms_source": "CUDA events over the timed region / filter launches in it",
                "kernel_ms_isolated": round(statistics.mean(per), 5),
                "kernel_ms_isolated_min": round(min(per), 5)}
    if prof.get("alu"):
        roofline["alu"] = {k: v for k, v in prof["alu"].items() if v is not None}
    alu = read_alu_floor(cfg.name)
    if alu:
        # the binding roofline for every config (ALU floor > HBM floor): ALU-pipe lane-ops per
        # pixel are a property of the kernel and the scene (counted from the ncu SASS mix of
        # the committed capture), the time is this run's per-launch kernel time
        ops = alu["alu_lane_ops_per_px"] * batch_px
        peak_alu = 64 * 148 * 1.965e9
        roofline.setdefault("alu", {}).update({
            "lane_ops_per_px": round(alu["alu_lane_ops_per_px"], 2),
            "achieved_Tops": round(ops / (kernel_ms * 1e-3) / 1e12, 3),
            "peak_Tops": round(peak_alu / 1e12, 3),
            "frac": round(ops / (kernel_ms * 1e-3) / peak_alu, 4),
            "floor_us": round(ops / peak_alu * 1e6, 2),
            "source": alu["source"]})
        if "instr_per_px" in alu:
            # issue roofline: every instruction needs an issue slot (4 per clk per SM)
            instr = alu["instr_per_px"] * batch_px
            peak_issue = 128 * 148 * 1.965e9
            roofline["issue"] = {"instr_per_px": round(alu["instr_per_px"], 2),
                                 "floor_us": round(instr / peak_issue * 1e6, 2),
                                 "frac": round(instr / (kernel_ms * 1e-3) / peak_issue, 4),
                                 "peak_Tinstr": round(peak_issue / 1e12, 3)}

    # e2e through the C-ABI host entry: pinned host in/out, H2D + filter + D2H each step
    e2e_steps = args.e2e_steps if args.e2e_steps is not None else max(3, min(steps, 20 if batch_bytes > (256 << 20) else 50))
    h_out = torch.empty_like(h_in).pin_memory()
    st = _native.IrdnStats()
    hfn = lib.irdn_run_filter_u8 if bpp == 1 else lib.irdn_run_filter_u16
    for _ in range(2):
        _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, 0, passes, local, ctypes.byref(st)))
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
    def e2e_run(mode: str):
        prev = _native.set_host_return(mode)
        try:
            _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, 0, passes, local,
                              ctypes.byref(st)))
            if world > 1:
                import torch.distributed as dist

                dist.barrier()
            t0 = time.perf_counter()
            for _ in range(e2e_steps):
                _native.check(hfn(h_in.data_ptr(), h_out.data_ptr(), B, H, W, cfg.k, 0, passes, local,
                                  ctypes.byref(st)))
            secs = time.perf_counter() - t0
            if world > 1:
                secs = _max_over_ranks(secs, dev)
            h2d, d2h = _native.last_transfer()
        finally:
            _native.set_host_return(prev)
        # consistency: the e2e output equals the device-resident output
        if not torch.equal(h_out.to(dev), outs[0]):
            raise AssertionError(f"e2e output ({mode} return) differs from the device-resident output")
        return world * batch_px * passes * e2e_steps / secs / 1e6, h2d, d2h

    full_v, _, full_d2h = e2e_run("full")
    e2e_v, h2d, d2h = e2e_run("auto")
    e2e = {"value": round(e2e_v, 3), "unit": "Mpix/s",
           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "steps": e2e_steps,
           "api": f"irdn_run_filter_{cfg.dtype} (C ABI, include/irdn.h) on pinned host buffers; "
                  "host wall clock, call is synchronous",
           "result_return": "sparse (changed pixels only, rebuilt on the host from its input; DESIGN.md §7.1)"
                            if d2h < batch_bytes else "full D2H copy (auto mode: 8-bit frames, or < 6 host "
                                                      "threads per GPU process; DESIGN.md §7.1)",
           "full_copy": {"value": round(full_v, 3), "d2h_bytes_per_step": full_d2h}}
    if st.detected * steps != det:
        raise AssertionError(f"counter mismatch: {st.detected}*{steps} != {det}")

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle

        oracle.lib()
        px, secs, desc = cpu_sample_run(cfg, host, 1, args.cpu_seconds)
        cpu = {"value": round(px / secs / 1e6, 4), "unit": "Mpix/s", "cores": 1, "kind": "port",
               "sample": desc + f" ({secs:.1f} s)",
               "note": "oracle/fnr_oracle.c (reference algorithm restated in C: clamp gather, "
                       "min/max detector, introsort median), single thread"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "Mpix/s", "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": round(ms_per_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype,
            "data": "synthetic (seeded IR scenes, DESIGN.md §5)",
            "config": {"workload": workload_desc(cfg), "frames_per_gpu": B, "height": H, "width": W,
                       "k": cfg.k, "method": "fnr", "passes": passes,
                       **({"multipass_launch": True} if args.multipass and passes > 1 else {}),
                       "detected_per_step": det // steps,
                       "l2": f"rotating {R} distinct in/out batch buffers "
                             f"({2 * R * batch_bytes / 1e6:.0f} MB > 2x L2)" if R > 1 else
                             f"in+out {2 * batch_bytes / 1e6:.0f} MB per step > 2x L2",
                       "launch": "CUDA graph of R launches" if graph is not None else "eager",
                       "parallelism": f"frame-sharded x{world}" if world > 1 else "1 GPU"},
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": gpu_launches, "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.path != "filter":
        import bench_aux

        return {"noise": bench_aux.run_noise, "sqerr": bench_aux.run_sqerr}[args.path](args, sys.modules[__name__])
    from paper_1201_3972_b200.scene import CONFIGS

    cfg = CONFIGS[args.config]
    world, rank, local = dist_setup(args.gpus)
    if args.impl == "reference":
        rc = run_reference_arm(args, cfg, rank, world)
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return rc
    return run_b200_arm(args, cfg, rank, world, local)


if __name__ == "__main__":
    sys.exit(main())
