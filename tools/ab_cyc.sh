#!/bin/bash
# Clock-independent A/B: ncu sm__cycles_elapsed.max of the attention kernel per variant and shape.
#   tools/ab_cyc.sh out.txt lib1 lib2 ...
out=$1; shift
cyc() {
  lib=$1; shift
  IG_LIB_OVERRIDE=$lib KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:attn_tc -s 6 -c 3 --csv python tools/kbench.py --which attn --iters 3 "$@" 2>/dev/null | grep -E "sm__cycles_elapsed" | awk -F'","' '{gsub(/"/,"",$NF); gsub(/,/,"",$NF); printf "%s ", $NF}'
  echo
}
for lib in "$@"; do
  echo -n "$lib flux2355: "; cyc $lib --qlens 2355
  echo -n "$lib flux1331: "; cyc $lib --qlens 1331
  echo -n "$lib unet819: "; cyc $lib --dh 64 --heads 10 --L 4096 --qlens 819
  echo -n "$lib unet4096: "; cyc $lib --dh 64 --heads 10 --L 4096 --qlens 4096
  echo -n "$lib unet1024: "; cyc $lib --dh 64 --heads 20 --L 1024 --qlens 1024
done > $out 2>&1
cat $out
