#!/bin/bash
# Run ON the GPU box: collect.sh + summaries, keeping gpurun_out/ under gpurun's 64 MiB
# copy-back limit (summaries and the c2 capture come back; the other .ncu-rep stay remote).
# usage: tools/prof/collect_remote.sh TAG [configs...]
cd "$(dirname "$0")/../.."
TAG=$1; shift
bash tools/prof/collect.sh $TAG "$@" > /dev/null 2>&1
python tools/prof/summarize.py gpurun_out/prof_$TAG $TAG > gpurun_out/prof_$TAG/summary.md 2>&1
python tools/prof/alu_floor.py gpurun_out/prof_$TAG $TAG > gpurun_out/prof_$TAG/alu_floor.log 2>&1
mkdir -p gpurun_out/prof_$TAG/profiles
cp profiles/*$TAG* profiles/ncu_summary.json gpurun_out/prof_$TAG/profiles/ 2>/dev/null
for f in gpurun_out/prof_$TAG/full_*.ncu-rep; do
  c=$(basename $f .ncu-rep)
  ncu -i $f --page source --csv --print-source cuda,sass > gpurun_out/prof_$TAG/src_$c.csv 2>/dev/null
  python tools/prof/cuda_lines.py gpurun_out/prof_$TAG/src_$c.csv 40 > gpurun_out/prof_$TAG/lines_$c.txt 2>&1
  rm -f gpurun_out/prof_$TAG/src_$c.csv
  [ "$c" = "full_c2" ] || rm -f $f
done
du -sh gpurun_out
