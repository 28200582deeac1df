mkdir -p gpurun_out
./tools/mma_ts_micro > gpurun_out/mma_ts_micro.txt 2>&1; echo "micro rc=$?"
R=r02
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1; echo "launches rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
      -o gpurun_out/${R}_ncu_tc_pair_rowdot python scripts/profile_module.py --steps 3 > /dev/null 2>&1; echo "ncu U rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_rowdot -s 2 -c 2 \
      -o gpurun_out/${R}_ncu_gram_and_v python scripts/profile_module.py --steps 3 > /dev/null 2>&1; echo "ncu GV rc=$?"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gram_reduce -s 1 -c 1 \
      -o gpurun_out/${R}_ncu_gram_reduce python scripts/profile_module.py --steps 3 > /dev/null 2>&1; echo "ncu red rc=$?"
ls -la gpurun_out
