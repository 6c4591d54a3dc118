set -x
cyc() {
  k=$1; shift
  KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:$k -s 3 -c 2 --csv python tools/kbench.py "$@" --iters 3 2>/dev/null | grep -E "sm__cycles_elapsed|tensor" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'
  echo
}
for e in "" "IG_GEMM_NO_BN160=1"; do
  for sh in "8192 1280 5120" "131072 320 2880" "32768 640 5760" "8192 1280 11520" "16384 2560 2560"; do set -- $sh
    echo -n "[$e] store $sh: "; env $e true; eval "$e cyc gemm_tc2 --which gemm --M $1 --N $2 --K $3"
  done
done > gpurun_out/r2c25_bn_ab.txt 2>&1
cat gpurun_out/r2c25_bn_ab.txt
