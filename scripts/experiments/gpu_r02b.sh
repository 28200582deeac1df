#!/bin/bash
# Round-2 re-entry check on one B200: GPU tests, smoke, default bench, and ncu captures of
# the norm's side-stream GEMMs (gram_tc = tc_rowdot<1>, gram_reduce, V = tc_rowdot<0>) and U.
mkdir -p gpurun_out
R=${1:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/${R}_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/${R}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/${R}_smoke.log
timeout 900 python bench.py > gpurun_out/${R}_bench_default.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${R}_bench_default.log | cut -c1-400
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${R}_launches.csv python scripts/profile_module.py --steps 3 --bwd > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"tc_rowdot|gram_reduce" -s 0 -c 3 \
    -o gpurun_out/${R}_ncu_side python scripts/profile_module.py --steps 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tc_pair_rowdot -s 1 -c 1 \
    -o gpurun_out/${R}_ncu_tc_pair_rowdot python scripts/profile_module.py --steps 3 > /dev/null 2>&1
ls gpurun_out
