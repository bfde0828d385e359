#!/bin/bash
# e2e (host buffers through irdn_run_filter_*) per config: sparse vs full result return.
# usage: tools/e2e_check.sh [configs...]   (run on the GPU box)
cd "$(dirname "$0")/.."
for c in ${@:-c2 c1 c3 c4 c5}; do
  python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 20 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$c', 'kernel', d['value'], 'e2e sparse', e['value'], 'd2h', e['d2h_bytes_per_step'], 'full', e['full_copy']['value'], 'd2h', e['full_copy']['d2h_bytes_per_step'])" 2>&1
done
