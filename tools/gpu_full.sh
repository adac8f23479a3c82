# round-end style run: smoke, gpu tests, bench (with CPU baseline), reference arm, launch list
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
nproc > gpurun_out/nproc.txt
timeout 900 python bench.py > gpurun_out/bench_full.log 2>gpurun_out/bench_full.err; echo "bench rc=$?" >> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>gpurun_out/bench_ref.err; echo "ref rc=$?" >> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_launch.log 2>&1
tail -n 2 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench_full.log gpurun_out/bench_ref.log gpurun_out/nproc.txt
