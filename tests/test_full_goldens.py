"""Full-size BASELINE configs vs full-size goldens (tests/golden/full_configs.json, made by
tests/golden/make_full_goldens.py from the oracle): sha256 of the whole output and the
FilterStats counters (FNR and MF), through the device path and (c2, c4 FNR) the host path
with the sparse result return. The input sha256 is checked first, so a scene-generator drift cannot pass
as a filter mismatch."""

import hashlib
import json
import os

import numpy as np
import pytest

import paper_1201_3972_b200 as P
from paper_1201_3972_b200.scene import CONFIGS, generate

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = json.load(open(os.path.join(HERE, "golden", "full_configs.json")))


def _sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_full_goldens_cover_every_config():
    assert {g["config"] for g in GOLD.values()} == {"c1", "c2", "c3", "c4", "c5"}


@pytest.mark.gpu
@pytest.mark.parametrize("key", sorted(GOLD))
def test_full_size_config_matches_golden(cuda_ok, key):
    import torch

    g = GOLD[key]
    cfg = CONFIGS[g["config"]]
    img = generate(cfg)
    assert list(img.shape) == g["shape"] and _sha(img) == g["input_sha256"]
    u16 = img.dtype == np.uint16
    t = torch.from_numpy(img.view(np.int16) if u16 else img).cuda()
    method = g.get("method", "fnr")
    out, st = P.run_filter(t.view(torch.uint16) if u16 else t, P.WindowSpec(g["k"]), method, g["passes"])
    host = (out.view(torch.int16) if u16 else out).cpu().numpy()
    host = host.view(np.uint16) if u16 else host
    assert _sha(host) == g["output_sha256"], key
    assert [st.minmax_scans, st.sorts, st.replacements, st.detected, st.passes] == g["stats"], key
    del t, out
    if g["config"] in ("c2", "c4") and method == "fnr":  # host buffers: pipelined copies + sparse return
        hout, hst = P.run_filter(img, P.WindowSpec(g["k"]), method, g["passes"])
        assert _sha(hout) == g["output_sha256"], key
        assert [hst.minmax_scans, hst.sorts, hst.replacements, hst.detected, hst.passes] == g["stats"], key
