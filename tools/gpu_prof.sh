# tests for the new scan, bench, launch list, full ncu capture of K1/K2/K4
timeout 900 python -m pytest tests/test_kpm_scan_gpu.py tests/test_engine_gpu.py -q --timeout 600 -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_synth|k1_analyze|k4_kpm" -s 3 -c 3 -o gpurun_out/prof_r1 python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/pytest_gpu.log gpurun_out/bench.log gpurun_out/ncu_full.log
