#!/bin/bash
# every runtime measurement switch must keep the norm / compose / fused-LoRA parity tests green
mkdir -p gpurun_out; O=gpurun_out/knob_parity.txt; : > $O
for kv in "DFX_PAIR_TMA3D=0" "DFX_PAIR_ZSMEM=0" "DFX_PAIR_KA=1" "DFX_PAIR_STAGES=3" "DFX_V_WIDE=1" "DFX_V_GSTAT=0" \
          "DFX_V_HALF=1" "DFX_V_PAIRS=16" "DFX_NORM_STRATEGY=0" "DFX_NORM_STRATEGY=2" "DFX_NORM_SIDE=28" "DFX_FIN_RESET=1" \
          "DFX_W_PREFETCH=2" "DFX_U_NH=2" "DFX_NORM_PAIR=0" "DFX_NORM_FUSE=0"; do
  r=$(env $kv timeout 600 python -m pytest tests/test_gpu_norm.py tests/test_gpu_vkernel.py -q -x -p no:cacheprovider 2>&1 | tail -1)
  echo "$kv | $r" >> $O
done
for kv in "DFX_BWD_CFG=4x2" "DFX_BWD_CFG=12x1" "DFX_LC_MIN_STAGES=2"; do
  r=$(env $kv timeout 600 python -m pytest tests/test_gpu_compose.py tests/test_gpu_lora_compose.py -q -x -p no:cacheprovider 2>&1 | tail -1)
  echo "$kv | $r" >> $O
done
cat $O
