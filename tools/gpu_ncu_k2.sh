timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_tc|k1_analyze|k4_kpm" -s 3 -c 3 -o gpurun_out/prof_tc python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_full.log 2>&1
tail -n 3 gpurun_out/ncu_full.log
