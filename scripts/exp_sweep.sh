#!/bin/bash
O=gpurun_out/exp.txt; : > $O
timeout 400 python -m pytest tests/test_gpu_norm.py -x -q > gpurun_out/t_norm.log 2>&1; echo "norm tests rc=$?" >> $O; tail -2 gpurun_out/t_norm.log >> $O
B="timeout 120 python bench.py --no-cpu-baseline --e2e-steps 0 --lora-steps 0 --variant-steps 0 --steps 800"
run() { echo "== $1" >> $O; shift; $B "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], {k:v['avg_us'] for k,v in d['kernels'].items()})" >> $O 2>&1; }
run base
for n in 96 80 72 64 48; do run sms$n --norm-sms $n; done
run infer64 --mode infer --norm-sms 64
run infer0 --mode infer
