for cfg in "" "DFX_NORM_PAIR=0" "DFX_EXP_NOCHAIN=1"; do
  echo "== $cfg"; env $cfg timeout 120 python bench.py --steps 500 --e2e-steps 0 --no-cpu-baseline 2>&1 | grep -o 'timed.*\|"[a-z_]*": {"launches_per_step[^}]*}' | sed 's/"bound.*share"/ share/' | cut -c1-110; done
