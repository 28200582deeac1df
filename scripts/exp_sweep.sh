#!/bin/bash
O=gpurun_out/exp.txt; : > $O
B="timeout 120 python bench.py --config c1 --mode infer --steps 200 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline"
for ns in 0 2 3 4 6; do
  echo "== ns $ns" >> $O
  if [ $ns = 0 ]; then $B 2>/dev/null; else DFX_F32_NS=$ns $B 2>/dev/null; fi | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k:v['avg_us'] for k,v in d['kernels'].items()})" >> $O 2>&1
done
