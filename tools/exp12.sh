timeout 600 python -m pytest tests/test_massive_mimo_gpu.py tests/test_pipeline_gpu.py tests/test_tx_packed.py tests/test_scene_gpu.py -q -x 2>&1 | tail -2
for args in "--n-ant 64 --layers 4 --slots 8" ""; do
timeout 300 python bench.py $args --steps 20 --warmup 5 --no-cpu-baseline --latency-slots 0 2>/dev/null | python -c "
import json,sys;d=json.loads(sys.stdin.read().strip().splitlines()[-1]);print('$args',round(d['value']),d['roofline']['kernel_ms'], round(d['roofline']['frac'],3), round(d['roofline']['step_frac'],3))"
done
