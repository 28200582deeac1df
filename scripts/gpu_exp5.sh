mkdir -p gpurun_out; O=gpurun_out/exp5.txt; : > $O
run() { env "$@" timeout 120 python scripts/exp_norm_prof.py --budget 104 --iters 20 --tag "$*" >> $O 2>&1; env "$@" timeout 120 python scripts/exp_norm_prof.py --budget 0 --iters 20 --tag "$*" >> $O 2>&1; }
run X=0
run DFX_Z_PREFETCH=1
run DFX_W_PREFETCH=2
run DFX_W_PREFETCH=6
run DFX_COMMIT_UMMAS=32 DFX_COMMIT_CAPDIV=1
run DFX_COMMIT_UMMAS=8
run DFX_COMMIT_UMMAS=32 DFX_COMMIT_CAPDIV=1 DFX_Z_PREFETCH=1
cat $O | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()); continue
    print(d['tag'].ljust(50), d['budget'], 'wall', d['norm_wall_us'], 'U', d.get('u_rowdot_tc'))
"
