"""Multi-GPU partitioning of the FNR pass: frame shards or row strips, no data-path collective.

The reference runs one process and splits rows into bands inside a thread pool
(pkg/src/irdenoise/filters.py:110-120: ``bounds = height * i // workers``),
merging per-band counters afterwards (:121-126). Here one process drives one
GPU and the same two decompositions are applied across ranks:

* a batch of frames is split into contiguous frame ranges (each rank filters
  whole frames; nothing crosses ranks);
* a single frame is split into row strips with the reference's band bounds;
  each rank reads its strip plus ``r * passes`` halo rows above and below
  (clamped to the frame) and filters with row clamping against the GLOBAL
  frame (irdn_filter_strip_*), so every output byte equals the one-GPU result.
  Multi-pass strips recompute the halo rows locally (over-fetch) instead of
  exchanging them between passes; the recomputed rows are not counted.

Only the FilterStats counters are reduced across ranks (one all_reduce of five
integers); outputs stay sharded unless ``gather=True``.
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
    """Frames across ranks when batch > 1, else row strips with r*passes halo rows."""
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
            plan.append(Shard(i, "rows", 0, 1, lo, hi, max(0, lo - halo), min(height, hi + halo)))
    return plan


# strip_fn(in_rows, in_row0, height, row_begin, row_end, k, method) -> (out_rows, detected, replaced)
StripFn = Callable[[np.ndarray, int, int, int, int, int, str], tuple]


def cuda_strip_fn(device: int = 0) -> StripFn:
    """Row-strip pass on `device` through the C ABI (irdn_filter_strip_{u8,u16})."""
    import torch

    from . import _native

    lib = _native.load_lib()

    def fn(in_rows: np.ndarray, in_row0: int, height: int, y0: int, y1: int, k: int, method: str):
        dev = torch.device("cuda", device)
        src = torch.from_numpy(np.ascontiguousarray(in_rows).view(np.int16 if in_rows.dtype == np.uint16 else np.uint8)).to(dev)
        out = torch.empty((y1 - y0, in_rows.shape[1]), dtype=src.dtype, device=dev)
        counts = torch.zeros(2, dtype=torch.int64, device=dev)
        f = lib.irdn_filter_strip_u8 if in_rows.dtype == np.uint8 else lib.irdn_filter_strip_u16
        with torch.cuda.device(dev):
            _native.check(f(src.data_ptr(), in_row0, in_rows.shape[0], out.data_ptr(), y0, y1, height,
                            in_rows.shape[1], in_rows.shape[1], in_rows.shape[1], k, _native.METHODS[method],
                            counts.data_ptr(), torch.cuda.current_stream(dev).cuda_stream))
            det, rep = (int(v) for v in counts.cpu().tolist())
        return out.cpu().numpy().view(in_rows.dtype), det, rep

    return fn


def filter_strip_passes(frame_rows: np.ndarray, shard: Shard, height: int, k: int, method: str, passes: int,
                        strip_fn: StripFn) -> tuple[np.ndarray, int, int]:
    """All passes of one row strip. frame_rows holds global rows [shard.in0, shard.in1).

    Pass p (0-based) produces rows [y0 - r*(P-1-p), y1 + r*(P-1-p)) clamped to the
    frame; only the owned rows [y0, y1) are counted, the halo extension is
    recomputed (with its counters discarded) so later passes see exact rows.
    """
    r = k // 2
    cur, cur0 = frame_rows, shard.in0
    det = rep = 0
    for p in range(passes):
        ext = r * (passes - 1 - p)
        a, b = max(0, shard.y0 - ext), min(height, shard.y1 + ext)
        parts = []
        for lo, hi, counted in ((a, shard.y0, False), (shard.y0, shard.y1, True), (shard.y1, b, False)):
            if hi <= lo:
                continue
            need0, need1 = max(0, lo - r), min(height, hi + r)
            sub = cur[need0 - cur0:need1 - cur0]
            o, d, rr = strip_fn(sub, need0, height, lo, hi, k, method)
            parts.append(o)
            if counted:
                det += d
                rep += rr
        cur, cur0 = np.concatenate(parts, axis=0), a
    return cur, det, rep


def run_shard(img: np.ndarray, shard: Shard, k: int, method: str, passes: int,
              strip_fn: StripFn) -> tuple[np.ndarray, list[int]]:
    """Filter this rank's shard of `img` ([B,H,W] or [H,W]). Returns (local output, counters)."""
    frames = img if img.ndim == 3 else img[None]
    _, height, width = frames.shape
    local_px = 0
    if shard.kind == "frames":
        outs, det, rep = [], 0, 0
        for f in range(shard.f0, shard.f1):
            o, d, rr = filter_strip_passes(frames[f], Shard(shard.rank, "rows", 0, 1, 0, height, 0, height),
                                           height, k, method, passes, strip_fn)
            outs.append(o)
            det += d
            rep += rr
        out = np.stack(outs) if outs else np.empty((0, height, width), frames.dtype)
        local_px = out.size
    else:
        out, det, rep = filter_strip_passes(frames[0][shard.in0:shard.in1], shard, height, k, method, passes,
                                            strip_fn)
        local_px = out.size
    if method == "fnr":
        counters = [local_px * passes, det, rep, det]
    else:
        counters = [0, local_px * passes, 0, 0]
    return out, counters


def run_filter_distributed(img: np.ndarray, k: int, method: str = "fnr", passes: int = 1, *,
                           group=None, gather: bool = True, strip_fn: StripFn | None = None):
    """run_filter over all ranks of `group` (torch.distributed, NCCL or gloo).

    Every rank passes the same `img` (or at least its own shard's rows); returns
    (output, FilterStats-like dict). With gather=True rank 0 receives the full
    image and the other ranks None; otherwise each rank keeps its shard.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    frames = img if img.ndim == 3 else img[None]
    plan = shard_plan(frames.shape[0], frames.shape[1], world, k, passes)
    shard = plan[rank]
    if strip_fn is None:
        strip_fn = cuda_strip_fn(torch.cuda.current_device())
    out, c = run_shard(img, shard, k, method, passes, strip_fn)
    t = torch.tensor(c, dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    dist.all_reduce(t, group=group)
    scans, sorts, rep, det = (int(v) for v in t.cpu().tolist())
    stats = {"minmax_scans": scans, "sorts": sorts, "replacements": rep, "detected": det, "passes": passes}
    if not gather:
        return out, stats
    parts = [None] * world if rank == 0 else None
    dist.gather_object(out, parts, dst=0, group=group)
    if rank != 0:
        return None, stats
    if shard.kind == "frames":
        full = np.concatenate([p for p in parts if p.size], axis=0)
    else:
        full = np.concatenate(parts, axis=0)[None]
    return (full if img.ndim == 3 else full[0]), stats
