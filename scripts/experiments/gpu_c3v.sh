#!/bin/bash
mkdir -p gpurun_out; O=gpurun_out/c3v.txt; : > $O
for cfg in c3 c4r64 c4r1024; do
for v in 0 1; do
  DFX_V_GSTAT=$v DFX_PLAN_PRINT=1 timeout 120 python scripts/exp_norm_prof.py --config $cfg --budget 0 --iters 10 --tag "gstat $v" 2>&1 | sort | uniq >> $O
done
done
DFX_V_GSTAT=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/c3_launches.csv python scripts/profile_module.py --config c3 --steps 2 > /dev/null 2>&1
grep -v "^==" gpurun_out/c3_launches.csv | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; ik=h.index('Kernel Name'); iv=h.index('Metric Value')
for x in r[1:]:
  if 'dfx' in x[ik]: print(x[ik][:60], x[iv])" >> $O
cat $O
