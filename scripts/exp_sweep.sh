for cfg in "DFX_NORM_PAIR=1" "DFX_NORM_PAIR=0" "DFX_NORM_PAIR=1" "DFX_NORM_PAIR=0"; do
  echo "== $cfg"; env $cfg timeout 120 python bench.py --steps 4000 --e2e-steps 0 --no-cpu-baseline --prof-steps 2 2>&1 | grep -o 'timed.*'; done
timeout 300 python bench.py > gpurun_out/bench6.json 2> gpurun_out/bench6.err; echo rc=$?; tail -3 gpurun_out/bench6.err | cut -c1-300
