# usage: tools/addsub_sweep.sh "lib tags" "configs"
for t in $1; do for c in $2; do
IRDN_LIB=build_variants/libirdn_$t.so python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$t', '$c', d['ms_per_step'], d['roofline']['kernel_ms_isolated'])"
done; done
