#!/bin/bash
# Run ON the GPU box: collect.sh for the given configs, then per config the ncu summary,
# CUDA-line and SASS-opcode histograms; keeps only the small text outputs.
# usage: tools/prof/collect_lines.sh TAG configs...
cd "$(dirname "$0")/../.."
TAG=$1; shift
bash tools/prof/collect.sh $TAG "$@" > /dev/null 2>&1
python tools/prof/summarize.py gpurun_out/prof_$TAG $TAG > gpurun_out/prof_$TAG/summary.md 2>&1
cp profiles/ncu_${TAG}_*.txt gpurun_out/prof_$TAG/ 2>/dev/null
for c in "$@"; do
  f=gpurun_out/prof_$TAG/full_$c.ncu-rep
  [ -f $f ] || continue
  ncu -i $f --page source --csv --print-source cuda,sass > /tmp/src_cs_$c.csv 2>/dev/null
  python tools/prof/cuda_lines.py /tmp/src_cs_$c.csv 50 > gpurun_out/prof_$TAG/lines_$c.txt 2>&1
  ncu -i $f --page source --csv --print-source sass > /tmp/src_s_$c.csv 2>/dev/null
  python tools/prof/sass_hist.py /tmp/src_s_$c.csv > gpurun_out/prof_$TAG/sass_$c.txt 2>&1
  rm -f $f
done
