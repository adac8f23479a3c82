O=gpurun_out
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_B.json 2> $O/bench_B.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --n-ant 64 --layers 4 --slots 8 --no-cpu-baseline --latency-slots 0 > $O/bench_E.json 2> $O/bench_E.err
timeout 900 python bench.py --cells 8 --layers 2 --slots 16 --no-cpu-baseline > $O/bench_C.json 2> $O/bench_C.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --latency-slots 0 > $O/ncu_launch.log 2>&1
tail -n 2 $O/smoke.log $O/pytest_gpu.log
