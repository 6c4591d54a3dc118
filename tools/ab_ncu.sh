#!/bin/bash
# A/B kernel durations measured by ncu (kernel time only, clocks unlocked):
#   tools/ab_ncu.sh <kernel-regex> "<kbench args>" lib1 lib2 ...
kre="$1"; args="$2"; shift 2
for lib in "$@"; do
  for r in 1 2; do
    IG_LIB_OVERRIDE=$lib IG_OP_REPEAT=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$kre -s 30 -c 20 --csv \
      python tools/kbench.py $args 2>/dev/null | grep gpu__time_duration | awk -F'","' -v L=$lib '{gsub(/"/,"",$NF); print L, $NF}' \
      | sort -k2 -n | awk '{a[NR]=$2; l=$1} END {print l, "median_us", a[int(NR/2)+1], "min_us", a[1], "n", NR}'
  done
done
