set -x
mkdir -p gpurun_out
cyc() {  # lib, kernel regex, kbench args...
  lib=$1; k=$2; shift 2
  IG_LIB_OVERRIDE=ablibs/$lib KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:$k -s 6 -c 4 --csv python tools/kbench.py "$@" --iters 3 2>/dev/null | grep -E "sm__cycles_elapsed" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'
  echo
}
for v in lib_gbase.so lib_gpipe.so; do
  for sh in "8192 1280 1280" "32768 640 640" "8192 1280 5120" "14720 3072 3072"; do set -- $sh; echo -n "$v gated $sh: "; cyc $v gemm_tc2 --which gated --M $1 --N $2 --K $3; done
done > gpurun_out/r2c17_gated_cyc.txt 2>&1
cat gpurun_out/r2c17_gated_cyc.txt
for v in lib_p128_0.so lib_p128_16.so; do
  echo -n "$v attn flux: "; cyc $v attn_tc --which attn
  echo -n "$v attn flux m0.2: "; cyc $v attn_tc --which attn --qlens 512,819
done > gpurun_out/r2c17_attn128_cyc.txt 2>&1
cat gpurun_out/r2c17_attn128_cyc.txt
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c17_unet_sweep_hbm.json > gpurun_out/r2c17_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c17_sweep.log | head -3
