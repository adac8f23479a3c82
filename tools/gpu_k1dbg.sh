timeout 900 python -m pytest tests -m gpu -q --timeout 600 -p no:cacheprovider -x 2>&1 | tail -3
ARCHES_K1P_DBG=1 timeout 300 python tools/profile_step.py --slots 256 --steps 3 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv python tools/profile_step.py --slots 256 --steps 3 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launches.csv
