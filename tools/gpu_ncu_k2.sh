timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k2_tc" -s 2 -c 1 -o gpurun_out/prof_k2 python tools/profile_step.py --slots 256 --steps 3 > gpurun_out/ncu_k2.log 2>&1
tail -2 gpurun_out/ncu_k2.log
