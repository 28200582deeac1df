#!/bin/bash
O=gpurun_out/exp.txt; : > $O
B="timeout 120 python bench.py --no-cpu-baseline --e2e-steps 0 --lora-steps 0 --variant-steps 0 --steps 2000"
run() { echo "== $*" >> $O; $B "$@" 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])" >> $O 2>&1; }
run --pipeline 8
run --pipeline 16
run --pipeline 40
run --pipeline 40 --nbuf 8
run --pipeline 16 --mode infer
run --pipeline 40 --mode infer
