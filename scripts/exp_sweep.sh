#!/bin/bash
O=gpurun_out/exp.txt; : > $O
for st in 4 8 10 12; do
  echo "== bwd stages $st" >> $O
  DFX_LIB=variants/libdfx_bwd$st.so timeout 60 python scripts/exp_kernels.py --what bwd --tag st$st >> $O 2>&1
  DFX_LIB=variants/libdfx_bwd$st.so timeout 120 python scripts/exp_green.py 72 80 bwd 2>&1 | tail -1 >> $O
  DFX_LIB=variants/libdfx_bwd$st.so timeout 120 python bench.py --no-cpu-baseline --e2e-steps 0 --lora-steps 0 --variant-steps 0 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('bench', d['value'], d['ms_per_step'])" >> $O 2>&1
done
timeout 60 python scripts/exp_kernels.py --what bwd,dual --tag st6 >> $O 2>&1
