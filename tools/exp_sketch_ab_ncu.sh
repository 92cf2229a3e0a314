#!/bin/bash
# A/B the tcgen05 sketch kernel between the in-tree library and an alternative
# build at base clocks (ncu --clock-control base), which removes the power-cap
# drift that dominates back-to-back event timings. Usage: LIB_B ell...
LIB_B=$1; shift
for ell in "$@"; do
  for v in A B; do
    if [ $v = B ]; then export SPIDGPU_LIB_PATH=$(realpath $LIB_B); else unset SPIDGPU_LIB_PATH; fi
    ncu --clock-control base --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg -k regex:sketch_tc_kernel \
      --csv python tools/exp_sketch_one.py $ell 2>/dev/null | grep -E 'gpu__time|sm__cycles' | \
      awk -F'","' -v v=$v -v ell=$ell '{gsub(/"/,"",$NF); printf "%s ell %s %s %s\n", v, ell, $(NF-2), $NF}'
  done
done
