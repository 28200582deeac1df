mkdir -p gpurun_out
for v in ${VARS:-base komma kochain koboth}; do
  for b in ${BUDGETS:-0 80}; do
    DFX_LIB=variants/libdfx_$v.so timeout 180 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tc_pair --csv python scripts/profile_module.py --steps 3 --budget $b 2>/dev/null | grep gpu__time_duration | awk -F'","' -v v=$v -v b=$b '{gsub(/"/,"",$NF); s=s" "$NF} END{print v, "budget", b, ":", s}'
  done
done
