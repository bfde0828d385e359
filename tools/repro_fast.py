"""Run one tile-kernel call per (dtype, k) and report the first failure (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1201_3972_b200 as P
from oracle import oracle
cases = [(np.uint8, 3, (9, 16)), (np.uint8, 3, (64, 256)), (np.uint16, 5, (64, 256)), (np.uint8, 7, (40, 160)),
         (np.uint16, 11, (70, 300)), (np.uint16, 9, (33, 64))]
only = sys.argv[1:] and int(sys.argv[1])
rng = np.random.default_rng(0)
for i, (dt, k, shape) in enumerate(cases):
    if only not in (0, None, []) and i != only - 1:
        continue
    img = rng.integers(0, 256 if dt == np.uint8 else 16384, shape).astype(dt)
    try:
        got, st = P.run_filter(img, P.WindowSpec(k), "fnr", 1)
    except Exception as e:
        print("FAIL", dt.__name__, k, shape, e); sys.exit(1)
    want, wst = oracle.run_filter_c(img, k, "fnr", 1)
    print(dt.__name__, k, shape, "equal" if np.array_equal(got, want) else "DIFF",
          [st.minmax_scans, st.sorts, st.replacements, st.detected], list(wst.counters())[:4])
