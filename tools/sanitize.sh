#!/bin/bash
# Run ON the GPU box: compute-sanitizer memcheck / racecheck / synccheck / initcheck over
# small instances of every kernel (tools/sanitize_cases.py), one process per tool x case.
# usage: tools/sanitize.sh TAG [cases...]    -> gpurun_out/sanitize_TAG/
cd "$(dirname "$0")/.."
TAG=$1; shift
CASES=${@:-warp multipass k3 large generic strip noise_metrics delta}
OUT=gpurun_out/sanitize_$TAG
mkdir -p $OUT
SUM=$OUT/summary.txt
: > $SUM
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check no"
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  for c in $CASES; do
    log=$OUT/${tool}_$c.log
    timeout 900 compute-sanitizer --tool $tool $extra --error-exitcode 9 --target-processes all \
      python tools/sanitize_cases.py $c > $log 2>&1
    rc=$?
    errs=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" $log | tail -1)
    echo "$tool $c rc=$rc $errs" | tee -a $SUM
  done
done
