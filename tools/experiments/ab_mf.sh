for r in 1 2; do for lib in base.so rows.so rows_alu.so rows_fin1.so; do for c in c5 c1; do
IRDN_LIB=build_variants/$lib python bench.py --config $c --method mf --steps 500 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', '$c', 'mf', d['ms_per_step'], d['roofline']['frac'])"
done; done; done
