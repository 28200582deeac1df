mkdir -p gpurun_out
O=gpurun_out/exp_commit.txt; : > $O
for b in 0 104; do for c in 4 8 16 24 32 48; do
  DFX_COMMIT_UMMAS=$c timeout 120 python scripts/exp_norm_prof.py --budget $b >> $O 2>&1
done; done
for cfg in c3 c1; do for c in 4 24; do
  DFX_COMMIT_UMMAS=$c timeout 120 python scripts/exp_norm_prof.py --config $cfg >> $O 2>&1
done; done
cat $O
timeout 900 python -m pytest tests/test_gpu_norm.py tests/test_gpu_dsplit.py tests/test_gpu_dist.py -q -x -p no:cacheprovider > gpurun_out/exp2_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/exp2_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 3 > gpurun_out/exp2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/exp2_bench.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['avg_us'], d['roofline'].get('unbudgeted'), d['roofline_norm_stage'], {k:v['avg_us'] for k,v in d['kernels'].items()}, d['variants']['infer']['value'])"
