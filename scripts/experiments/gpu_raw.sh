#!/bin/bash
mkdir -p gpurun_out/ko
echo "PYTORCH_CUDA_ALLOC_CONF=$PYTORCH_CUDA_ALLOC_CONF" > gpurun_out/ko/raw.txt
python scripts/profile_module.py --steps 1 --raw-alloc >> gpurun_out/ko/raw.txt 2>&1
for v in "" "--raw-alloc"; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_pair_rowdot" --csv \
     --log-file gpurun_out/ko/raw_$([ -z "$v" ] && echo torch || echo cuda).csv python scripts/profile_module.py --steps 3 $v > /dev/null 2>&1
done
