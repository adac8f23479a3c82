timeout 600 python -m pytest tests/test_kpm_scan_gpu.py tests/test_engine_gpu.py tests/test_benched_shape_gpu.py tests/test_switch_properties_gpu.py -q -x 2>&1 | tail -3
timeout 300 python bench.py --n-prb 52 --policy tree --slots 1024 --steps 20 --warmup 5 --no-cpu-baseline --latency-slots 0 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('A',round(d['value']),d['roofline']['kernel_ms'], d['roofline']['frac'], d['roofline']['step_frac'])"
timeout 300 python bench.py --mode policy-stress --steps 50 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('D',round(d['value']),d['us_per_boundary'])"
