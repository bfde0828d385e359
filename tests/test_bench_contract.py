"""bench.py output contract (the driver parses its last stdout line as JSON).

CPU: the reference arm (`--impl reference`, the oracle port on host cores).
GPU: the B200 arm (default filter path, `--passes 2`, the widened rows `--path`).
"""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=REPO)
    assert out.returncode == 0, out.stderr[-2000:]
    line = out.stdout.strip().splitlines()[-1]
    return json.loads(line)


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1"])
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Mpix/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["config"]["workload"].startswith("c1")
    # the reference arm's config block is the B200 arm's (the driver compares them)
    import bench
    from paper_1201_3972_b200.scene import CONFIGS

    assert d["config"] == bench.config_block(CONFIGS["c1"], 1, 1)


def test_default_workload_is_the_largest_single_gpu_config():
    import bench
    from paper_1201_3972_b200.scene import CONFIGS

    sys.argv = ["bench.py"]
    assert bench.parse().config == "c5"
    assert max(CONFIGS.values(), key=lambda c: c.pixels).name == "c5"


def test_work_split_follows_the_survey_plan():
    """c2/c3/c5 split frames, c4 row strips with r-row halos, c1 replicas."""
    import bench
    from paper_1201_3972_b200.scene import CONFIGS

    for name in ("c2", "c3", "c5"):
        cfg = CONFIGS[name]
        for n in (1, 2, 4, 8):
            shares = [bench.rank_share(cfg, n, r) for r in range(n)]
            assert [s["f0"] for s in shares] == [cfg.frames * r // n for r in range(n)]
            assert sum(s["f1"] - s["f0"] for s in shares) == cfg.frames
    c4 = CONFIGS["c4"]
    for n in (2, 4, 8):
        shares = [bench.rank_share(c4, n, r) for r in range(n)]
        assert shares[0]["in0"] == 0 and shares[-1]["in1"] == c4.height
        assert sum(s["y1"] - s["y0"] for s in shares) == c4.height
        for s in shares:
            assert s["kind"] == "rows" and s["y0"] - s["in0"] <= 5 and s["in1"] - s["y1"] <= 5
    assert bench.rank_share(CONFIGS["c1"], 4, 3)["replica"]
    assert bench.scaling_kind(CONFIGS["c1"], 4) == "weak" and bench.scaling_kind(c4, 4) == "strong"


@pytest.mark.gpu
def test_b200_arm_line(cuda_ok):
    d = _run(["--steps", "50", "--warmup", "3", "--cpu-seconds", "1"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["config"]["workload"].startswith("c5") and d["dtype"] == "u8"
    assert d["roofline"]["static_ops"]["minmax_instr_per_px"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 50
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]


@pytest.mark.gpu
def test_b200_arm_passes2_and_widened_rows(cuda_ok):
    d = _run(["--config", "c2", "--steps", "20", "--warmup", "3", "--passes", "2", "--no-cpu-baseline"])
    assert d["config"]["passes"] == 2 and d["gpu_launches"] >= 40
    for path in ("noise", "sqerr"):
        d = _run(["--path", path, "--steps", "10", "--warmup", "3", "--cpu-seconds", "1"])
        assert BASE_KEYS <= set(d) and d["value"] > 0 and d["roofline"]["unit"] == "GB/s"
        assert d["cpu_baseline"]["value"] > 0 and d["e2e"]["value"] > 0


def test_reference_arm_under_torchrun_world2():
    """Launched like the driver does for N > 1: rank 0 alone prints the line, the other
    rank exits 0 without work; the config block names the N-GPU split."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "c2", "--steps", "1", "--warmup", "1",
           "--ref-seconds", "0.5"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["parallelism"].startswith("frame-sharded over 2 GPUs")


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["c4", "c2"])
def test_b200_arm_under_torchrun_world2(cuda_ok, config):
    """Code-path check of the N-GPU split on a 1-GPU box (both ranks share the GPU, gloo
    control plane): c4 as two row strips with halos, c2 as two frame shards; one line
    from rank 0 with the separately timed gather. Not a scaling measurement."""
    import socket

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(REPO, "bench.py"),
           "--gpus", "2", "--config", config, "--steps", "20", "--warmup", "3", "--e2e-steps", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=REPO)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["gather"]["bytes"] == d["run"]["pixels_per_step"] * (2 if d["dtype"] == "u16" else 1)
    if config == "c4":
        assert d["run"]["rank0_share"]["kind"] == "rows" and d["run"]["rank0_share"]["y1"] == 4096
        assert d["config"]["parallelism"].startswith("row strips over 2 GPUs")
    else:
        assert d["run"]["rank0_share"] == {"kind": "frames", "f0": 0, "f1": 32, "replica": False}
    assert d["e2e"]["value"] > 0
