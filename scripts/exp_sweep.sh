#!/bin/bash
O=gpurun_out/exp.txt; : > $O
E="timeout 60 python scripts/exp_kernels.py"
for sv in 8 7 6 4 2; do DFX_BWD_SV=$sv $E --what bwd --tag sv$sv >> $O 2>&1; done
for sv in 8 7 4; do DFX_BWD_SV=$sv $E --config c1 --what bwd --tag sv$sv >> $O 2>&1; done
