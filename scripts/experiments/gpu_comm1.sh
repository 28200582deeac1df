#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_comm.py tests/test_gpu_dist.py tests/test_gpu_dsplit.py -q -p no:cacheprovider 2>&1 | tail -1
for ar in dfx nccl; do
  timeout 600 python bench.py --mode dsplit --allreduce $ar --steps 20 --warmup 5 > gpurun_out/r02_dsplit_$ar.log 2>&1; echo "dsplit $ar rc=$? $(tail -1 gpurun_out/r02_dsplit_$ar.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["exchange_us"])')"
done
