timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --latency-slots 0 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('B',round(d['value']),d['roofline']['kernel_ms'], d['roofline']['frac'])"
