"""Full-size goldens for the five BASELINE configs (SURVEY §8c "Full-size goldens").

The reference itself is far too slow at these sizes (k = 11 u16 at ~0.015 Mpix/s), so the
outputs come from the C restatement of its algorithm (oracle/fnr_oracle.c, pinned to the
reference on every shape class by tests/test_oracle_golden.py), run over the full seeded
scenes (paper_1201_3972_b200/scene.py). Stored per config: sha256 of the output bytes and
the FilterStats counters; the GPU test (tests/test_full_goldens.py) reproduces both.

    python tests/golden/make_full_goldens.py      # writes tests/golden/full_configs.json
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)

from oracle import oracle  # noqa: E402
from paper_1201_3972_b200.scene import CONFIGS, generate  # noqa: E402

CASES = [("c1", 1, "fnr"), ("c2", 1, "fnr"), ("c2", 2, "fnr"), ("c3", 1, "fnr"), ("c4", 1, "fnr"), ("c5", 1, "fnr"),
         ("c1", 1, "mf"), ("c2", 1, "mf"), ("c3", 1, "mf"), ("c4", 1, "mf"), ("c5", 1, "mf")]


def main() -> None:
    threads = len(os.sched_getaffinity(0))
    out = {}
    cache = {}
    for name, passes, method in CASES:
        cfg = CONFIGS[name]
        t0 = time.perf_counter()
        img = cache[name] if name in cache else generate(cfg)
        cache = {name: img}
        res, st = oracle.run_filter_c(img, cfg.k, method, passes, threads=threads)
        key = f"{name}_{method}_p{passes}"
        out[key] = {
            "config": name, "k": cfg.k, "method": method, "passes": passes, "shape": list(img.shape),
            "dtype": str(img.dtype),
            "input_sha256": hashlib.sha256(img.tobytes()).hexdigest(),
            "output_sha256": hashlib.sha256(res.tobytes()).hexdigest(),
            "stats": [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes],
        }
        print(key, out[key]["stats"], f"{time.perf_counter() - t0:.1f} s", flush=True)
    with open(os.path.join(HERE, "full_configs.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()
