#!/bin/bash
# lora_compose A/B: variants/libdfx_<name>.so against the HEAD kernel (variants/libdfx_old.so);
# a name of the form NAME@ENV=VAL runs variant NAME with that environment setting
VARS=${@:-old bias ahead4b}
for rep in 1 2; do for v in $VARS; do
  n=${v%%@*}; envs=""; [ "$n" != "$v" ] && envs=${v#*@}
  env $envs DFX_LIB=variants/libdfx_$n.so timeout 300 python scripts/lc_bench.py $v 2>&1 | grep outs | grep -v unsupported
done; done
