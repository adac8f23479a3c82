# round evidence: smoke, GPU tests, bench (B, with CPU baseline), reference arm,
# configs C and E bench lines, bench launch list, ncu full capture of K1/K2/K3/K4
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt; nproc >> gpurun_out/smi.txt
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_B.json 2> gpurun_out/bench_B.err; echo "bench rc=$?" >> gpurun_out/bench_B.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 python bench.py --streams 16 --slots 16 --steps 30 --warmup 3 --no-cpu-baseline --latency-slots 0 > gpurun_out/bench_C.json 2> gpurun_out/bench_C.err
timeout 900 python bench.py --n-ant 64 --streams 4 --slots 8 --steps 20 --warmup 3 --no-cpu-baseline --latency-slots 0 > gpurun_out/bench_E.json 2> gpurun_out/bench_E.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/bench_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --latency-slots 0 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc|k2_tc|k3_fin|k4_kpm" -s 5 -c 5 -o gpurun_out/prof_full python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_full.log 2>&1
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench_B.json gpurun_out/bench_ref.json gpurun_out/bench_C.json gpurun_out/bench_E.json | cut -c1-300
