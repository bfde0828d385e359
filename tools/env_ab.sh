#!/bin/bash
# A/B of environment settings on the device-resident bench (kernel ms per step).
# usage: tools/env_ab.sh "VAR=a VAR=b ..." "c2 c4" reps
for r in $(seq ${3:-3}); do for e in $1; do for c in $2; do
env $e python bench.py --config $c --steps 500 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$e', '$c', d['ms_per_step'], d['roofline']['kernel_ms_isolated'])"
done; done; done
