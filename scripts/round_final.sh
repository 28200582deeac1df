#!/bin/bash
# Round-end evidence on one B200 (under gpurun): GPU tests, smoke, bench (both arms),
# the bench's ncu launch list, and the ncu full captures (scripts/round_profile.sh).
R=${1:-r01}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/${R}_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/${R}_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${R}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/${R}_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/${R}_bench.log > gpurun_out/${R}_bench_c2.json
timeout 600 python bench.py --impl reference > gpurun_out/${R}_bench_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/${R}_bench_ref.log > gpurun_out/${R}_bench_reference_c2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/${R}_bench_launches_raw.csv python bench.py --steps 40 --warmup 3 --no-cpu-baseline --e2e-steps 1 --lora-steps 2 --variant-steps 40 > /dev/null 2>&1
echo "bench launch list rc=$?"
bash scripts/round_profile.sh $R
ls gpurun_out | grep $R
