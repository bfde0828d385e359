#!/bin/bash
# Run ON the GPU box: one bench line per BASELINE config (fnr and mf), the default line and
# the reference arm, into gpurun_out/sweep_TAG/.  usage: tools/bench_sweep.sh TAG
cd "$(dirname "$0")/.."
TAG=$1
OUT=gpurun_out/sweep_$TAG
mkdir -p $OUT
timeout 600 python bench.py > $OUT/default.json 2> $OUT/default.err
timeout 600 python bench.py --impl reference > $OUT/reference.json 2> $OUT/reference.err
for c in c1 c2 c3 c4 c5; do
  timeout 300 python bench.py --config $c --no-cpu-baseline > $OUT/fnr_$c.json 2> $OUT/fnr_$c.err
  timeout 300 python bench.py --config $c --method mf --no-cpu-baseline --e2e-steps 2 > $OUT/mf_$c.json 2> $OUT/mf_$c.err
done
timeout 300 python bench.py --config c5 --passes 2 --no-cpu-baseline --e2e-steps 2 > $OUT/fnr_c5_p2.json 2> $OUT/fnr_c5_p2.err
OUT=$OUT python - <<'PY' > $OUT/table.md
import json, glob, os
print("| line | Mpix/s | ms/step | HBM frac | e2e Mpix/s | static min/max instr/px |")
print("|---|---|---|---|---|---|")
for f in sorted(glob.glob(os.environ.get("OUT", "gpurun_out/sweep_x") + "/*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception:
        continue
    rf = d.get("roofline", {})
    print(f"| {os.path.basename(f)[:-5]} | {d.get('value')} | {d.get('ms_per_step')} | {rf.get('frac')} | "
          f"{(d.get('e2e') or {}).get('value')} | {(rf.get('static_ops') or {}).get('minmax_instr_per_px')} |")
PY
