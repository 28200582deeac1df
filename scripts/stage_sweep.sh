#!/bin/bash
# Stage analysis of the pipelined training step: each stage alone and the norm SM budget.
# usage: scripts/stage_sweep.sh "ONLY_LIST" "NORM_SMS_LIST"
for only in ${1:-both norm compose}; do
  o=$only; [ "$o" = both ] && o=""
  for ns in ${2:-64 80 96}; do
    out=$(timeout 200 python bench.py --no-cpu-baseline --e2e-steps 0 --lora-steps 0 --variant-steps 0 --prof-steps 4 --steps 800 ${o:+--only $o} --norm-sms $ns 2>&1 | tail -1)
    v=$(echo "$out" | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'])" 2>/dev/null || echo "FAILED: ${out:0:300}")
    echo "only=$only norm_sms=$ns: $v"
  done
done
