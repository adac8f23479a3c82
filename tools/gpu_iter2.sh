timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --latency-slots 200 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_tc|k1_analyze|k4_kpm" -s 3 -c 3 -o gpurun_out/prof_tc python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench.log
