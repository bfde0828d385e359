# usage: tools/tail_sweep.sh "tail values" "ovkeep values" "configs"
for tw in ${1:-1}; do for ok in ${2:-256}; do for c in ${3:-c2}; do
  IRDN_TAIL=$tw IRDN_OVKEEP=$ok python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('tail $tw ovkeep $ok', '$c', d['roofline']['kernel_ms'], d['ms_per_step'])"
done; done; done
