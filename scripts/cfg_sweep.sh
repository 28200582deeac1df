#!/bin/bash
# value + per-kernel times for each config (analysis helper); extra args go to bench.py
O=${SWEEP_OUT:-gpurun_out/sweep.txt}; : > $O
for cfg in c2 c3 c4r64 c4r128 c4r512 c4r1024 c1; do
  for mode in train infer; do
    timeout 300 python bench.py --config $cfg --mode $mode --steps 400 --e2e-steps 0 --lora-steps 0 --variant-steps 0 --no-cpu-baseline "$@" > /tmp/c.json 2>/tmp/c.err || { echo "$cfg $mode failed" >> $O; tail -3 /tmp/c.err >> $O; continue; }
    python -c "
import json; d=json.load(open('/tmp/c.json'))
print('$cfg', '$mode', round(d['value'],1), 'modules/s', round(d['ms_per_step']*1e3,1), 'us/step', {n:v['avg_us'] for n,v in d['kernels'].items()})" >> $O
  done
done
