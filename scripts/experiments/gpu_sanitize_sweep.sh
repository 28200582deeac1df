#!/bin/bash
# compute-sanitizer on every kernel (both V kernels) + every config in both modes + C5.
mkdir -p gpurun_out; O=gpurun_out/r02_sanitize.txt; : > $O
for v in 0 1; do
  DFX_V_GSTAT=$v timeout 600 compute-sanitizer --tool memcheck python scripts/sanitize.py > gpurun_out/san_mem_$v.log 2>&1
  echo "memcheck DFX_V_GSTAT=$v rc=$? $(grep -E 'ERROR SUMMARY|sanitize run ok' gpurun_out/san_mem_$v.log | tr '\n' ' ')" >> $O
done
DFX_V_GSTAT=1 timeout 900 compute-sanitizer --tool synccheck python scripts/sanitize.py > gpurun_out/san_sync.log 2>&1
echo "synccheck rc=$? $(grep -E 'ERROR SUMMARY|sanitize run ok' gpurun_out/san_sync.log | tr '\n' ' ')" >> $O
DFX_V_GSTAT=1 timeout 1200 compute-sanitizer --tool racecheck python scripts/sanitize.py > gpurun_out/san_race.log 2>&1
echo "racecheck rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize run ok' gpurun_out/san_race.log | tr '\n' ' ')" >> $O
cat $O
SWEEP_OUT=gpurun_out/r02_config_sweep.txt bash scripts/cfg_sweep.sh
for mode in train infer; do
  timeout 600 python bench.py --config c5 --mode $mode --steps 3 --warmup 3 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline > /tmp/c5.json 2>/tmp/c5.err
  echo "c5 $mode $(tail -1 /tmp/c5.json | cut -c1-200)" >> gpurun_out/r02_config_sweep.txt
done
cat gpurun_out/r02_config_sweep.txt
