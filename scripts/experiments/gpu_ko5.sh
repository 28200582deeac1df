#!/bin/bash
mkdir -p gpurun_out/ko
run() { tag=$1; shift; env "$@" timeout 300 ncu --metrics gpu__time_duration.sum,gpc__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"tc_pair_rowdot|tc_rowdot|gstat" --csv \
     --log-file gpurun_out/ko/$tag.csv python scripts/profile_module.py --steps 3 > /dev/null 2>&1; }
run fix_base X=0
run fix_ka1 DFX_PAIR_KA=1
run fix_skel_ka2 DFX_LIB=variants/libdfx_ko_allc.so
run fix_skel_ka1 DFX_PAIR_KA=1 DFX_LIB=variants/libdfx_ko_allc.so
run fix_komma DFX_LIB=variants/libdfx_ko_mma.so
for b in 0 140; do timeout 120 python scripts/exp_norm_prof.py --budget $b --iters 20 --tag fix >> gpurun_out/ko/fix_live.txt 2>&1; done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-cpu-full-module --e2e-steps 0 --lora-steps 0 --variant-steps 400 > gpurun_out/ko/fix_bench.log 2>&1
tail -1 gpurun_out/ko/fix_bench.log | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print("train", d["value"], "infer", d["variants"]["infer"]["value"], "U", d["roofline"]["avg_us"], d["roofline"]["frac"])' >> gpurun_out/ko/fix_live.txt
