# full check: smoke, GPU tests, bench, launch list, ncu full capture of K1/K2/K4
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --latency-slots 200 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_tc|k1_analyze|k4_kpm" -s 3 -c 3 -o gpurun_out/prof_full python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench.log
