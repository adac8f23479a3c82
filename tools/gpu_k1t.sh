python tools/k1_compare.py --n-prb 273 --slots 8 2>&1 | tail -4
python tools/k1_compare.py --n-prb 12 --slots 4 2>&1 | tail -4
timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -15
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/prof_step.log 2>&1
tail -3 gpurun_out/prof_step.log
python tools/launch_summary.py gpurun_out/launches.csv
