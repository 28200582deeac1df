#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_compose.py -q -x -p no:cacheprovider 2>&1 | tail -1
B="--steps 40 --warmup 20 --no-cpu-baseline --no-cpu-full-module --lora-steps 0 --variant-steps 0 --e2e-steps 0"
for rep in 1 2; do for v in nofmul2 head; do
  L=$([ $v = head ] && echo paper_2603_22276_b200/libdfx.so || echo variants/libdfx_$v.so)
  DFX_LIB=$L timeout 300 python scripts/exp_kernels.py --what bwd --iters 30 2>&1 | tail -1 | sed "s/^/$v alone: /"
  DFX_LIB=$L timeout 300 python bench.py $B > /tmp/k.log 2>&1; echo "$v step | $(tail -1 /tmp/k.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["kernels"]["compose_bwd_dmag"]["avg_us"])')"
done; done
