#!/bin/bash
# Run ON the GPU box: per BASELINE config, a plain bench run (exit 0 required), the ncu
# launch list of the same command, and one `--set full` capture of the filter kernel.
# usage: tools/prof/collect.sh TAG [configs...]
cd "$(dirname "$0")/../.."
TAG=$1; shift
CFGS=${@:-c1 c2 c3 c4 c5}
mkdir -p gpurun_out/prof_$TAG
for c in $CFGS; do
  CMD="python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --no-graph"
  $CMD > gpurun_out/prof_$TAG/bench_$c.json 2> gpurun_out/prof_$TAG/bench_$c.err || continue
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$TAG/launches_$c.csv $CMD > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:fnr_ -s 3 -c 1 \
      -o gpurun_out/prof_$TAG/full_$c $CMD > gpurun_out/prof_$TAG/ncu_$c.log 2>&1
done
ls -la gpurun_out/prof_$TAG
