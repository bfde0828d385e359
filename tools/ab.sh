# usage: tools/ab.sh "libA libB" "configs" reps
for r in $(seq ${3:-3}); do for lib in $1; do for c in $2; do
IRDN_LIB=build_variants/$lib python bench.py --config $c --steps 500 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', d['ms_per_step'], d['roofline']['kernel_ms_isolated'])"
done; done; done
