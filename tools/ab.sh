#!/bin/bash
# A/B kernel benchmark on the same box: tools/ab.sh "<kbench args>" lib1 lib2 ...
args="$1"; shift
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active,utilization.gpu --format=csv,noheader -lms 500 > gpurun_out/ab_clocks.csv &
SMI=$!
for r in 1 2 3 4; do for lib in "$@"; do echo -n "$lib: "; IG_LIB_OVERRIDE=$lib python tools/kbench.py $args; done; done
kill $SMI
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv
