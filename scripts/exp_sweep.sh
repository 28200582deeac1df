for cfg in "" "DFX_NORM_BA=after"; do
  for st in norm module; do echo "== $cfg $st"; env $cfg timeout 120 python bench.py --steps 2000 --e2e-steps 0 --no-cpu-baseline --prof-steps 2 --stage $st 2>&1 | grep -o 'timed.*'; done; done
