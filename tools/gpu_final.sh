# Final round evidence on one B200: smoke, GPU suite, bench lines (B default = packed tx, B complex,
# reference arm, C, E, A), the launch list of the headline bench, ncu --set full of K1 / K2 (config B).
O=gpurun_out
timeout 300 python __graft_entry__.py > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/smoke.log
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 900 python bench.py > $O/bench_B.json 2> $O/bench_B.err
timeout 900 python bench.py --tx complex --no-cpu-baseline > $O/bench_Bc.json 2> $O/bench_Bc.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 python bench.py --n-prb 52 --policy tree --slots 1024 --no-cpu-baseline > $O/bench_A.json 2> $O/bench_A.err
timeout 900 python bench.py --cells 8 --layers 2 --slots 16 --no-cpu-baseline > $O/bench_C.json 2> $O/bench_C.err
timeout 900 python bench.py --n-ant 64 --layers 4 --slots 8 --no-cpu-baseline --latency-slots 0 > $O/bench_E.json 2> $O/bench_E.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --latency-slots 0 > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc|k2_tc|k1_tc_finalize" -s 3 -c 3 -o $O/prof_B -f python tools/profile_step.py --slots 256 --steps 3 --tx packed > $O/ncu_B.log 2>&1
tail -n 2 $O/smoke.log $O/pytest_gpu.log
