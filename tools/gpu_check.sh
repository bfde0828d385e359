#!/bin/bash
# Round-trip helper run ON the GPU box: parity tests, then a short bench per config.
# usage: tools/gpu_check.sh [configs...]   (default: c2 c1 c3 c4 c5)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -m pytest tests -x -q -m gpu 2>&1 | tail -4
CFGS=${@:-c2 c1 c3 c4 c5}
for c in $CFGS; do
  python bench.py --config $c --steps 100 --warmup 3 --no-cpu-baseline --e2e-steps 3 2>&1 | tail -1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'][:2], 'value', d['value'], 'Mpix/s  kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'e2e', d['e2e']['value'], 'clk', d['clocks'].get('sm_mhz'))" 2>&1
done
