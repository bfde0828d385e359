#!/bin/bash
# A/B of library variants with extra bench flags.  usage: ab_any.sh "libA.so libB.so" "c3 c2" "--method mf" reps
for r in $(seq ${4:-2}); do for lib in $1; do for c in $2; do
IRDN_LIB=build_variants/$lib python bench.py --config $c $3 --steps 300 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', '$3', d['ms_per_step'], d['roofline']['frac'])"
done; done; done
