mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/g1_smi.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/g1_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/g1_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/g1_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/g1_bench_s20.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/g1_bench_s20.log
