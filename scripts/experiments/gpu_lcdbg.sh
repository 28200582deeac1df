#!/bin/bash
for lib in paper_2603_22276_b200/libdfx.so variants/libdfx_lcdep.so variants/libdfx_lcfence.so variants/libdfx_lcboth.so variants/libdfx_lcold.so; do
  echo "== $lib"; DFX_LIB=$lib timeout 100 python scripts/lc_debug.py 2>&1 | grep mismatches
done
