#!/bin/bash
# e2e (host-buffer training step) vs the number of row chunks in dfx_module_train_host
for c in ${1:-4 8 16 32}; do
  v=$(DFX_E2E_CHUNKS=$c timeout 200 python bench.py --no-cpu-baseline --e2e-steps 20 --lora-steps 0 --variant-steps 0 --prof-steps 4 --steps 400 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['value'])")
  echo "chunks=$c: e2e $v modules/s"
done
