# usage: tools/variants.sh "lib1 lib2 ..." "c2 c4"
for lib in $1; do for c in $2; do
  IRDN_LIB=$lib python bench.py --config $c --steps 50 --warmup 3 --no-cpu-baseline --e2e-steps 1 2>/dev/null | tail -1 | \
  python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib'.split('/')[-1], d['config']['workload'][:2], d['roofline']['kernel_ms'])"
done; done
