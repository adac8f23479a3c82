timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k1_tc" -s 2 -c 2 -o gpurun_out/prof_k1t python tools/profile_step.py --slots 256 --steps 2 > gpurun_out/ncu_k1.log 2>&1
tail -2 gpurun_out/ncu_k1.log
