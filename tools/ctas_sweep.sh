for n in 5 6 7 8 9 10; do for c in c2 c3 c4; do
IRDN_WARP_CTAS=$n python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas $n', '$c', d['roofline']['kernel_ms'], d['ms_per_step'])"
done; done
