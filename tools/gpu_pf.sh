for pf in 0 1 2 3 4; do
  ARCHES_K2_PREFETCH=$pf timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --latency-slots 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('pf', $pf, round(d['value']), d['roofline']['kernel_ms'])"
done
