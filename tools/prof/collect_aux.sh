#!/bin/bash
# Run ON the GPU box: the widened rows (bench.py --path noise|sqerr): plain bench run
# (exit 0 required), ncu launch list of the same command, one --set full capture.
# usage: tools/prof/collect_aux.sh TAG
cd "$(dirname "$0")/../.."
TAG=$1
mkdir -p gpurun_out/prof_$TAG
for path in noise sqerr; do
  case $path in noise) K=noise_kernel; STEPS=50;; sqerr) K=sq_err_kernel; STEPS=100;; esac
  CMD="python bench.py --path $path --steps $STEPS --warmup 3 --cpu-seconds 3"
  $CMD > gpurun_out/prof_$TAG/bench_$path.json 2> gpurun_out/prof_$TAG/bench_$path.err || continue
  ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file gpurun_out/prof_$TAG/launches_$path.csv $CMD > /dev/null 2>&1
  ncu --set full --clock-control none --import-source on -k regex:$K -s 5 -c 1 \
      -o gpurun_out/prof_$TAG/full_$path $CMD > gpurun_out/prof_$TAG/ncu_$path.log 2>&1
done
ls -la gpurun_out/prof_$TAG
