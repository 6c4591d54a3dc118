set -x
mkdir -p gpurun_out
cyc() {
  lib=$1; k=$2; shift 2
  IG_LIB_OVERRIDE=ablibs/$lib KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:$k -s 6 -c 3 --csv python tools/kbench.py "$@" --iters 3 2>/dev/null | grep -E "sm__cycles_elapsed" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'
  echo
}
for v in lib_a_base.so lib_a_st2.so lib_a_st4.so lib_a_p8.so lib_a_max3.so; do
  echo -n "$v flux: "; cyc $v attn_tc --which attn
  echo -n "$v flux m0.2: "; cyc $v attn_tc --which attn --qlens 512,819
  echo -n "$v unet l1: "; cyc $v attn_tc --which attn --dh 64 --heads 10 --L 4096 --qlens 4096 --nreq 8
done > gpurun_out/r2c22_attn_ab.txt 2>&1
cat gpurun_out/r2c22_attn_ab.txt
timeout 900 python tools/unet_full_sweep.py --tier host --depth 10 --ms 0.01,0.2,0.5 --out gpurun_out/r2c22_unet_host_d10.json > gpurun_out/r2c22_sweep_host_d10.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c22_sweep_host_d10.log
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 0 -c 40 -o gpurun_out/r2c22_unet_dense_gemms python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
