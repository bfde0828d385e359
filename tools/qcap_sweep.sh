for lib in build_variants/libirdn_q512.so build_variants/libirdn_q1024.so; do for n in 10 11 12 13 14; do
IRDN_LIB=$lib IRDN_WARP_CTAS=$n python bench.py --config c2 --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', 'ctas $n', d['roofline']['kernel_ms'], d['ms_per_step'])"
done; done
