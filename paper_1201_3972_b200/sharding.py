"""Multi-GPU partitioning of the filter: frame shards or row strips, no data-path collective.

The reference runs one process and splits rows into bands inside a thread pool
(pkg/src/irdenoise/filters.py:110-120: ``bounds = height * i // workers``) and merges
per-band counters afterwards (:121-126). Here one process drives one GPU and the same
decomposition is applied across ranks:

* a batch of frames is split into contiguous frame ranges (band bounds over frames);
  each rank filters its frames with ONE device call (irdn_run_filter_device_*);
* a single frame is split into row strips with the reference's band bounds; each rank
  holds its strip plus ``r * passes`` halo rows above and below (clamped to the frame)
  and filters with row clamping against the GLOBAL frame (irdn_filter_strip_*), so
  every output byte equals the one-GPU result. Multi-pass strips recompute the halo
  rows locally (over-fetch) instead of exchanging them between passes; the recomputed
  rows are not counted (`strip_pass_plan`).

Shards are device-resident: one host->device copy of the shard when the input is a
host array, the passes on the device, the output left on the device. The FilterStats
counters are all-gathered (four integers per rank) and summed on the host — no
reduction collective. With ``gather=True`` rank 0 receives every shard through one
``torch.distributed.gather`` (NCCL: peer transfers over NVLink; gloo: through the host).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np


@dataclass(frozen=True)
class Shard:
    """What one rank owns: frames [f0, f1), output rows [y0, y1), input rows [in0, in1)."""

    rank: int
    kind: str  # "frames" | "rows"
    f0: int
    f1: int
    y0: int
    y1: int
    in0: int
    in1: int


def band_bounds(n: int, parts: int) -> list[int]:
    """The reference's band bounds, ``n * i // parts`` (filters.py:116)."""
    parts = max(1, min(parts, n))
    return [n * i // parts for i in range(parts + 1)]


def shard_plan(batch: int, height: int, world: int, k: int, passes: int = 1) -> list[Shard]:
    """Frames across ranks when batch > 1, else row strips with r*passes halo rows. Ranks
    beyond the number of frames / rows get an empty shard."""
    if world < 1:
        raise ValueError("world must be >= 1")
    r = k // 2
    plan = []
    if batch > 1:
        b = band_bounds(batch, world)
        for i in range(world):
            lo, hi = (b[i], b[i + 1]) if i < len(b) - 1 else (batch, batch)
            plan.append(Shard(i, "frames", lo, hi, 0, height, 0, height))
    else:
        b = band_bounds(height, world)
        for i in range(world):
            lo, hi = (b[i], b[i + 1]) if i < len(b) - 1 else (height, height)
            halo = r * passes
            in0, in1 = (max(0, lo - halo), min(height, hi + halo)) if hi > lo else (lo, lo)
            plan.append(Shard(i, "rows", 0, 1, lo, hi, in0, in1))
    return plan


@dataclass(frozen=True)
class StripCall:
    """One strip-kernel call: output rows [row_begin, row_end) from input rows [need0, need1)."""

    row_begin: int
    row_end: int
    counted: bool  # the shard's own rows (halo recomputation is not counted)
    need0: int
    need1: int


def strip_pass_plan(shard: Shard, height: int, k: int, passes: int) -> list[tuple[int, int, list[StripCall]]]:
    """Per pass p (0-based): the rows it produces, [y0 - r*(P-1-p), y1 + r*(P-1-p)) clamped to
    the frame, as (a, b, calls). Pass p reads pass p-1's rows; only [y0, y1) is counted."""
    r = k // 2
    out = []
    if shard.y1 <= shard.y0:
        return out
    for p in range(passes):
        ext = r * (passes - 1 - p)
        a, b = max(0, shard.y0 - ext), min(height, shard.y1 + ext)
        calls = []
        for lo, hi, counted in ((a, shard.y0, False), (shard.y0, shard.y1, True), (shard.y1, b, False)):
            if hi > lo:
                calls.append(StripCall(lo, hi, counted, max(0, lo - r), min(height, hi + r)))
        out.append((a, b, calls))
    return out


# ---------------------------------------------------------------------------
# Host executor (numpy rows + a pluggable strip filter): the plan's CPU check
# ---------------------------------------------------------------------------
# strip_fn(in_rows, in_row0, height, row_begin, row_end, k, method) -> (out_rows, detected, replaced)
StripFn = Callable[[np.ndarray, int, int, int, int, int, str], tuple]


def filter_strip_passes(frame_rows: np.ndarray, shard: Shard, height: int, k: int, method: str, passes: int,
                        strip_fn: StripFn) -> tuple[np.ndarray, int, int]:
    """All passes of one row strip on the host. frame_rows holds global rows [shard.in0, shard.in1)."""
    cur, cur0 = frame_rows, shard.in0
    det = rep = 0
    for a, _, calls in strip_pass_plan(shard, height, k, passes):
        parts = []
        for c in calls:
            o, d, rr = strip_fn(cur[c.need0 - cur0:c.need1 - cur0], c.need0, height, c.row_begin, c.row_end, k,
                                method)
            parts.append(o)
            if c.counted:
                det += d
                rep += rr
        cur, cur0 = np.concatenate(parts, axis=0), a
    if shard.y1 <= shard.y0:
        return np.empty((0, frame_rows.shape[1]), frame_rows.dtype), 0, 0
    return cur, det, rep


def _counters(method: str, pixels: int, passes: int, det: int, rep: int) -> list[int]:
    """[minmax_scans, sorts, replacements, detected] as the reference counts them (filters.py:121-126)."""
    if method == "fnr":
        return [pixels * passes, det, rep, det]
    return [0, pixels * passes, 0, 0]


def run_shard(img: np.ndarray, shard: Shard, k: int, method: str, passes: int,
              strip_fn: StripFn) -> tuple[np.ndarray, list[int]]:
    """Filter this rank's shard of `img` ([B,H,W] or [H,W]) on the host executor."""
    frames = img if img.ndim == 3 else img[None]
    _, height, width = frames.shape
    if shard.kind == "frames":
        outs, det, rep = [], 0, 0
        for f in range(shard.f0, shard.f1):
            whole = Shard(shard.rank, "rows", 0, 1, 0, height, 0, height)
            o, d, rr = filter_strip_passes(frames[f], whole, height, k, method, passes, strip_fn)
            outs.append(o)
            det += d
            rep += rr
        out = np.stack(outs) if outs else np.empty((0, height, width), frames.dtype)
    else:
        out, det, rep = filter_strip_passes(frames[0][shard.in0:shard.in1], shard, height, k, method, passes,
                                            strip_fn)
    return out, _counters(method, out.size, passes, det, rep)


# ---------------------------------------------------------------------------
# Device executor (the product path: libirdn.so, one call per shard / strip call)
# ---------------------------------------------------------------------------
def run_shard_device(src, shard: Shard, height: int, k: int, method: str, passes: int, stream=None,
                     dst_ptr: int | None = None):
    """Filter a device-resident shard. `src` is a CUDA tensor of the shard's frames
    [f1-f0, H, W] or its input rows [in1-in0, W] (uint8, or uint16 / int16 bit patterns).
    Returns (device output, counters); the output stays on the device. With `dst_ptr` (a
    device pointer, possibly another GPU's memory mapped through CUDA IPC: the fused
    gather) the shard's final output is written there instead and the returned tensor is
    None."""
    import torch

    from . import _native

    lib = _native.load_lib()
    u16 = src.element_size() == 2
    t = "u16" if u16 else "u8"
    dev = src.device
    counts = torch.zeros(2, dtype=torch.int64, device=dev)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    m = _native.METHODS[method]
    width = src.shape[-1]
    with torch.cuda.device(dev):
        if shard.kind == "frames":
            nfr = shard.f1 - shard.f0
            out = torch.empty((nfr, height, width), dtype=src.dtype, device=dev) if dst_ptr is None else None
            if nfr:
                tmp = torch.empty((nfr, height, width), dtype=src.dtype, device=dev) if passes > 1 else None
                fn = getattr(lib, f"irdn_run_filter_device_{t}")
                _native.check(fn(src.data_ptr(), out.data_ptr() if out is not None else dst_ptr,
                                 tmp.data_ptr() if tmp is not None else None, nfr,
                                 height, width, k, m, passes, counts.data_ptr(), s.cuda_stream))
        else:
            fn = getattr(lib, f"irdn_filter_strip_{t}")
            junk = torch.zeros(2, dtype=torch.int64, device=dev)
            cur, cur0 = src, shard.in0
            out = torch.empty((0, width), dtype=src.dtype, device=dev)
            plan = strip_pass_plan(shard, height, k, passes)
            for pi, (a, b, calls) in enumerate(plan):
                last = pi == len(plan) - 1
                out = torch.empty((b - a, width), dtype=src.dtype, device=dev) if not (last and dst_ptr) else None
                for c in calls:
                    if out is not None:
                        dst = out[c.row_begin - a:].data_ptr()
                    else:  # the last pass produces exactly the owned rows [y0, y1)
                        dst = dst_ptr + (c.row_begin - shard.y0) * width * src.element_size()
                    _native.check(fn(cur[c.need0 - cur0:].data_ptr(), c.need0, c.need1 - c.need0, dst,
                                     c.row_begin, c.row_end, height, width, width, width, k, m,
                                     (counts if c.counted else junk).data_ptr(), s.cuda_stream))
                cur, cur0 = out, a
        det, rep = (int(v) for v in counts.tolist())  # the one host sync of the shard
    if shard.kind == "frames":
        npx = (shard.f1 - shard.f0) * height * width
    else:
        npx = max(0, shard.y1 - shard.y0) * width
    return out, _counters(method, npx, passes, det, rep)


def _gather_to_rank0(local, world: int, rank: int, group, backend: str):
    """One torch.distributed.gather of every rank's (flattened, padded) shard to rank 0."""
    import torch
    import torch.distributed as dist

    elem = local.dtype
    flat = local.reshape(-1).view(torch.uint8)  # bytes: gloo has no 16-bit integer collectives
    on_dev = backend == "nccl"
    n = torch.tensor([flat.numel()], dtype=torch.int64, device=flat.device if on_dev else "cpu")
    sizes = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(x.item()) for x in sizes]
    send = flat if on_dev else flat.cpu()
    mx = max(sizes)
    if send.numel() < mx:
        send = torch.cat([send, send.new_zeros(mx - send.numel())])
    bufs = [torch.empty_like(send) for _ in range(world)] if rank == 0 else None
    dist.gather(send, bufs, dst=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:sz] for b, sz in zip(bufs, sizes)]).view(elem)


def run_filter_distributed(img, k: int, method: str = "fnr", passes: int = 1, *,
                           group=None, gather: bool | str = True, strip_fn: StripFn | None = None):
    """run_filter over all ranks of `group` (torch.distributed, NCCL or gloo).

    `img` is a numpy array ([H,W] or [B,H,W], uint8 / uint16; every rank passes the same
    array, or at least its own shard's frames / rows) or a CUDA tensor of that shape.
    Returns (output, FilterStats-like dict). With gather=True rank 0 receives the full
    result (same kind as the input: numpy or tensor) and the other ranks None; otherwise
    every rank keeps its shard (on its GPU). gather="fused": rank 0's output buffer is
    mapped into every rank (CUDA IPC, irdn_ipc_*) and each rank's filter kernels store their
    shard's output straight into it over NVLink — the gather happens inside the filter
    launch, tile by tile, instead of as a collective afterwards. `strip_fn` swaps the
    device executor for the host one (CPU tests of the decomposition).
    """
    import torch
    import torch.distributed as dist

    if method not in ("fnr", "mf"):
        raise ValueError(f"unknown method {method!r}, expected 'fnr' or 'mf'")
    if passes < 1:
        raise ValueError(f"passes must be >= 1, got {passes}")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    is_tensor = type(img).__module__.startswith("torch")
    orig = img
    if is_tensor and img.dtype == torch.uint16:
        img = img.view(torch.int16)  # 16-bit pixels travel as int16 bit patterns
    ndim = img.ndim
    shape3 = tuple(img.shape) if ndim == 3 else (1, *img.shape)
    batch, height, width = shape3
    plan = shard_plan(batch, height, world, k, passes)
    shard = plan[rank]
    if strip_fn is not None:
        host = img.cpu().numpy() if is_tensor else img
        local, c = run_shard(host, shard, k, method, passes, strip_fn)
        local_t = torch.from_numpy(np.ascontiguousarray(local).view(np.int16 if local.dtype == np.uint16 else local.dtype))
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
        frames = img if ndim == 3 else img[None]
        part = frames[shard.f0:shard.f1] if shard.kind == "frames" else frames[0, shard.in0:shard.in1]
        if is_tensor:
            src = part.to(dev).contiguous()
        else:
            a = np.ascontiguousarray(part)
            src = torch.from_numpy(a.view(np.int16) if a.dtype == np.uint16 else a).to(dev)
        if gather == "fused":
            return _run_fused_gather(src, shard, shape3, ndim, k, method, passes, rank, world, group, backend,
                                     is_tensor, orig, img)
        local_t, c = run_shard_device(src, shard, height, k, method, passes)
    tot = torch.tensor(c, dtype=torch.int64, device=local_t.device if backend == "nccl" else "cpu")
    allc = [torch.empty_like(tot) for _ in range(world)]
    dist.all_gather(allc, tot, group=group)  # counters: gathered, summed on the host (no reduction)
    scans, sorts, rep, det = (int(v) for v in torch.stack(allc).cpu().sum(0).tolist())
    stats = {"minmax_scans": scans, "sorts": sorts, "replacements": rep, "detected": det, "passes": passes}
    u16 = (img.dtype == np.uint16) if not is_tensor else orig.dtype == torch.uint16
    if not gather:
        return local_t, stats
    full = _gather_to_rank0(local_t, world, rank, group, backend)
    if full is None:
        return None, stats
    full = full.reshape(shape3)
    if ndim == 2:
        full = full[0]
    if is_tensor:
        return full.to(orig.device).view(orig.dtype), stats
    a = full.cpu().numpy()
    return (a.view(np.uint16) if u16 else a), stats


def _run_fused_gather(src, shard: Shard, shape3, ndim: int, k: int, method: str, passes: int, rank: int,
                      world: int, group, backend: str, is_tensor: bool, orig, img):
    """The filter writes every rank's shard straight into rank 0's output (CUDA IPC)."""
    import ctypes

    import torch
    import torch.distributed as dist

    from . import _native

    lib = _native.load_lib()
    batch, height, width = shape3
    dev = src.device
    bpp = src.element_size()
    full = torch.empty(shape3, dtype=src.dtype, device=dev) if rank == 0 else None
    msg = [None]
    if rank == 0:
        handle = ctypes.create_string_buffer(64)
        off = ctypes.c_uint64(0)
        _native.check(lib.irdn_ipc_export(full.data_ptr(), handle, ctypes.byref(off)))
        msg = [(handle.raw, int(off.value))]
    dist.broadcast_object_list(msg, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    raw, off = msg[0]
    if rank == 0:
        base = full.data_ptr()
    else:
        ptr = ctypes.c_void_p()
        _native.check(lib.irdn_ipc_open(ctypes.create_string_buffer(raw, 64), off, ctypes.byref(ptr)))
        base = ptr.value
    try:
        if shard.kind == "frames":
            dst = base + shard.f0 * height * width * bpp
        else:
            dst = base + shard.y0 * width * bpp
        _, c = run_shard_device(src, shard, height, k, method, passes, dst_ptr=dst)
        torch.cuda.synchronize(dev)  # this rank's stores into rank 0's memory are complete
        dist.barrier(group=group)
    finally:
        if rank != 0:
            lib.irdn_ipc_close(ctypes.c_void_p(base), off)
    tot = torch.tensor(c, dtype=torch.int64, device=dev if backend == "nccl" else "cpu")
    allc = [torch.empty_like(tot) for _ in range(world)]
    dist.all_gather(allc, tot, group=group)
    scans, sorts, rep, det = (int(v) for v in torch.stack(allc).cpu().sum(0).tolist())
    stats = {"minmax_scans": scans, "sorts": sorts, "replacements": rep, "detected": det, "passes": passes}
    if rank != 0:
        return None, stats
    out = full if ndim == 3 else full[0]
    if is_tensor:
        return out.to(orig.device).view(orig.dtype), stats
    a = out.cpu().numpy()
    return (a.view(np.uint16) if img.dtype == np.uint16 else a), stats
