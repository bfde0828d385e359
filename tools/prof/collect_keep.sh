#!/bin/bash
# Run ON the GPU box: collect.sh for the given configs, plus CUDA-line and SASS-opcode
# histograms; keeps the .ncu-rep captures (mind gpurun's 64 MiB copy-back: ~25 MB each)
# so that tools/prof/summarize.py can be run on them here.  usage: collect_keep.sh TAG configs...
cd "$(dirname "$0")/../.."
TAG=$1; shift
bash tools/prof/collect.sh $TAG "$@" > /dev/null 2>&1
for c in "$@"; do
  f=gpurun_out/prof_$TAG/full_$c.ncu-rep
  [ -f $f ] || continue
  ncu -i $f --page source --csv --print-source cuda,sass > /tmp/src_cs_$c.csv 2>/dev/null
  python tools/prof/cuda_lines.py /tmp/src_cs_$c.csv 50 > gpurun_out/prof_$TAG/lines_$c.txt 2>&1
  ncu -i $f --page source --csv --print-source sass > /tmp/src_s_$c.csv 2>/dev/null
  python tools/prof/sass_hist.py /tmp/src_s_$c.csv > gpurun_out/prof_$TAG/sass_$c.txt 2>&1
done
ls -la gpurun_out/prof_$TAG
