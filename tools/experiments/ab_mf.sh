#!/bin/bash
# A/B of library variants on the MF method (tools/ab.sh runs FNR).
# usage: tools/experiments/ab_mf.sh "libA.so libB.so" "c5 c1" reps
for r in $(seq ${3:-2}); do for lib in $1; do for c in $2; do
IRDN_LIB=build_variants/$lib python bench.py --config $c --method mf --steps 500 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', 'mf', d['ms_per_step'], d['roofline']['frac'])"
done; done; done
