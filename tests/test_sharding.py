"""Multi-GPU decomposition (frame shards / row strips) — host logic on CPU with gloo, kernels on GPU.

The CPU tests plug the C oracle in as the per-strip filter, so the partitioning,
halo over-fetch, multi-pass recomputation and counter reduction are checked
without a GPU; the GPU test runs the same plan through irdn_filter_strip_*.
"""

import os
import socket

import numpy as np
import pytest

from oracle import oracle
from paper_1201_3972_b200 import sharding
from paper_1201_3972_b200.scene import CONFIGS, generate


def oracle_strip_fn(in_rows, in_row0, height, y0, y1, k, method):
    """Stand-in for the GPU strip kernel: rows outside the strip are poisoned, so any read
    beyond the halo the plan fetched would change the output."""
    frame = np.full((height, in_rows.shape[1]), 0xAB, dtype=in_rows.dtype)
    frame[in_row0:in_row0 + in_rows.shape[0]] = in_rows
    out, (det, rep) = oracle.filter_rows_c(frame, k, y0, y1, method)
    if method == "mf":
        det = rep = 0
    return out, det, rep


def test_band_bounds_match_reference_formula():
    for n in (1, 5, 17, 8192):
        for parts in (1, 2, 3, 8):
            b = sharding.band_bounds(n, parts)
            assert b[0] == 0 and b[-1] == n
            assert all(b[i] <= b[i + 1] for i in range(len(b) - 1))
            w = max(1, min(parts, n))
            assert b == [n * i // w for i in range(w + 1)]


def test_strip_pass_plan_reads_only_fetched_rows():
    """Every strip call of every pass reads rows the previous pass (or the fetched
    strip) holds, produces a contiguous range, and counts exactly the owned rows."""
    for height in (1, 7, 61):
        for world in (1, 2, 3, 8, 70):
            for k in (3, 5, 11):
                for passes in (1, 2, 3):
                    plan = sharding.shard_plan(1, height, world, k, passes)
                    assert sum(sh.y1 - sh.y0 for sh in plan) == height
                    for sh in plan:
                        have = (sh.in0, sh.in1)
                        for a, b, calls in sharding.strip_pass_plan(sh, height, k, passes):
                            assert [c.row_begin for c in calls][0] == a and calls[-1].row_end == b
                            assert all(x.row_end == y.row_begin for x, y in zip(calls, calls[1:]))
                            assert sum(c.row_end - c.row_begin for c in calls if c.counted) == sh.y1 - sh.y0
                            for c in calls:
                                assert have[0] <= c.need0 and c.need1 <= have[1], (height, world, k, passes, sh)
                            have = (a, b)
                        if sh.y1 > sh.y0:
                            assert have == (sh.y0, sh.y1)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8, 70])
@pytest.mark.parametrize("k,passes,method", [(5, 1, "fnr"), (11, 1, "fnr"), (3, 2, "fnr"), (5, 2, "mf")])
def test_row_strips_reassemble_exactly(world, k, passes, method):
    cfg = CONFIGS["c4"].with_shape(height=61, width=47)
    img = generate(cfg, nframes=1)[0]
    want, st = oracle.run_filter_c(img, k, method, passes)
    plan = sharding.shard_plan(1, img.shape[0], world, k, passes)
    parts, tot = [], np.zeros(4, dtype=np.int64)
    for sh in plan:
        out, c = sharding.run_shard(img, sh, k, method, passes, oracle_strip_fn)
        parts.append(out)
        tot += c
    assert np.array_equal(np.concatenate(parts), want)
    assert list(tot) == [st.minmax_scans, st.sorts, st.replacements, st.detected]


def test_frame_shards_reassemble_exactly():
    cfg = CONFIGS["c2"].with_shape(frames=5, height=23, width=31)
    img = generate(cfg, nframes=5)
    want, st = oracle.run_filter_c(img, 5, "fnr", 2)
    for world in (1, 2, 4, 8):
        parts, tot = [], np.zeros(4, dtype=np.int64)
        for sh in sharding.shard_plan(5, 23, world, 5, 2):
            out, c = sharding.run_shard(img, sh, 5, "fnr", 2, oracle_strip_fn)
            parts.append(out)
            tot += c
        assert np.array_equal(np.concatenate(parts), want)
        assert list(tot) == [st.minmax_scans, st.sorts, st.replacements, st.detected]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg, batch, k, method, passes = case
        scene = CONFIGS[cfg].with_shape(frames=batch, height=37, width=29)
        img = generate(scene, nframes=batch)
        if batch == 1:
            img = img[0]
        out, stats = sharding.run_filter_distributed(img, k, method, passes, strip_fn=oracle_strip_fn)
        q.put((rank, None if out is None else out.tobytes(), stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [("c4", 1, 11, "fnr", 1), ("c1", 1, 3, "fnr", 2), ("c2", 3, 5, "fnr", 1),
                                  ("c3", 1, 7, "mf", 1)])
def test_gloo_world2_matches_single_process(case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, case, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=180) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, batch, k, method, passes = case
    scene = CONFIGS[cfg].with_shape(frames=batch, height=37, width=29)
    img = generate(scene, nframes=batch)
    want, st = oracle.run_filter_c(img if batch > 1 else img[0], k, method, passes)
    by_rank = {r: (o, s) for r, o, s in res}
    assert by_rank[1][0] is None
    assert by_rank[0][0] == want.tobytes()
    for r in (0, 1):
        s = by_rank[r][1]
        assert [s["minmax_scans"], s["sorts"], s["replacements"], s["detected"], s["passes"]] == list(st.counters())


@pytest.mark.gpu
def test_gpu_device_shards_match_whole_frame(cuda_ok):
    """The device executor (one H2D per shard, strip calls / one frame call on the GPU,
    output left on the device) reassembles the single-GPU result for every rank count."""
    import torch

    import paper_1201_3972_b200 as P

    dev = torch.device("cuda", 0)
    cfg = CONFIGS["c4"].with_shape(height=1031, width=1280)
    img = generate(cfg, nframes=1)[0]
    for k, passes, method in ((11, 1, "fnr"), (11, 2, "fnr"), (5, 3, "mf")):
        whole, st = P.run_filter(img, P.WindowSpec(k), method, passes)
        for world in (2, 3, 8):
            parts, tot = [], np.zeros(4, dtype=np.int64)
            for sh in sharding.shard_plan(1, img.shape[0], world, k, passes):
                src = torch.from_numpy(np.ascontiguousarray(img[sh.in0:sh.in1]).view(np.int16)).to(dev)
                out, c = sharding.run_shard_device(src, sh, img.shape[0], k, method, passes)
                parts.append(out.cpu().numpy().view(np.uint16))
                tot += c
            assert np.array_equal(np.concatenate(parts), whole), (k, passes, world)
            assert list(tot) == [st.minmax_scans, st.sorts, st.replacements, st.detected]
    frames = generate(CONFIGS["c5"].with_shape(frames=7, height=96, width=128), nframes=7)
    whole, st = P.run_filter(frames, P.WindowSpec(3), "fnr", 2)
    parts, tot = [], np.zeros(4, dtype=np.int64)
    for sh in sharding.shard_plan(7, 96, 3, 3, 2):
        out, c = sharding.run_shard_device(torch.from_numpy(frames[sh.f0:sh.f1]).to(dev), sh, 96, 3, "fnr", 2)
        parts.append(out.cpu().numpy())
        tot += c
    assert np.array_equal(np.concatenate(parts), whole)
    assert list(tot) == [st.minmax_scans, st.sorts, st.replacements, st.detected]


def _cuda_worker(rank, world, port, case, q, gather=True):
    import torch
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)  # both ranks share the one GPU here
    try:
        torch.cuda.set_device(0)
        cfg, batch, k, method, passes, h, w = case
        scene = CONFIGS[cfg].with_shape(frames=batch, height=h, width=w)
        img = generate(scene, nframes=batch)
        if batch == 1:
            img = img[0]
        out, stats = sharding.run_filter_distributed(img, k, method, passes, gather=gather)  # CUDA strips / frames
        q.put((rank, None if out is None else out.tobytes(), stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("gather", [True, "fused"])
@pytest.mark.parametrize("case", [("c4", 1, 11, "fnr", 2, 700, 640), ("c2", 6, 5, "fnr", 1, 256, 320),
                                  ("c3", 1, 7, "mf", 1, 300, 512), ("c5", 5, 3, "fnr", 2, 120, 160)])
def test_gpu_world2_run_filter_distributed(cuda_ok, case, gather):
    """Two ranks (spawned processes, gloo control plane) filtering their row strips /
    frame shards with the CUDA kernels reassemble exactly the single-process result —
    gathered afterwards (torch.distributed.gather) or fused: rank 1's kernels store into
    rank 0's output through a CUDA IPC mapping (both ranks share the one GPU here, which
    exercises the same path as NVLink peers)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cuda_worker, args=(r, 2, port, case, q, gather)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    cfg, batch, k, method, passes, h, w = case
    scene = CONFIGS[cfg].with_shape(frames=batch, height=h, width=w)
    img = generate(scene, nframes=batch)
    want, st = oracle.run_filter_c(img if batch > 1 else img[0], k, method, passes)
    by_rank = {r: (o, s) for r, o, s in res}
    assert by_rank[1][0] is None and by_rank[0][0] == want.tobytes()
    s = by_rank[0][1]
    assert [s["minmax_scans"], s["sorts"], s["replacements"], s["detected"], s["passes"]] == list(st.counters())
