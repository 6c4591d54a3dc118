cyc() {
  lib=$1; shift
  IG_LIB_OVERRIDE=$lib KB_WARM=0.3 timeout 300 ncu --metrics sm__cycles_elapsed.max,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tc -s 3 -c 2 --csv python tools/kbench.py --which gemm --iters 3 "$@" 2>/dev/null | grep -E "sm__" | awk -F'","' '{gsub(/"/,"",$NF); gsub(/,/,"",$NF); printf "%s ", $NF}'
  echo
}
for lib in ablibs/lib_gbase.so ablibs/lib_gnarrow.so; do
  echo -n "$lib 131072x320x2880: "; cyc $lib --M 131072 --N 320 --K 2880
  echo -n "$lib 32768x640x5760: "; cyc $lib --M 32768 --N 640 --K 5760
  echo -n "$lib 8192x320x1280: "; cyc $lib --M 8192 --N 320 --K 1280
done
