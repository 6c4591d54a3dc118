set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c20_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c20_pytest.log
cyc() {
  lib=$1; k=$2; shift 2
  IG_LIB_OVERRIDE=ablibs/$lib KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:$k -s 6 -c 3 --csv python tools/kbench.py "$@" --iters 3 2>/dev/null | grep -E "sm__cycles_elapsed" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'
  echo
}
for v in lib_gred.so lib_tmast.so; do
  echo -n "$v store 14720x3072x3072: "; cyc $v gemm_tc2 --which gemm --M 14720 --N 3072 --K 3072
  echo -n "$v gelu 14720x12288x3072: "; cyc $v gemm_tc2 --which gemm --M 14720 --N 12288 --K 3072 --epi 1 --bias
  echo -n "$v store 8192x1280x1280: "; cyc $v gemm_tc --which gemm --M 8192 --N 1280 --K 1280
  echo -n "$v store 3000x3072x3072: "; cyc $v gemm_tc --which gemm --M 3000 --N 3072 --K 3072
done > gpurun_out/r2c20_store_cyc.txt 2>&1
cat gpurun_out/r2c20_store_cyc.txt
for v in lib_gred.so lib_tmast.so; do
  IG_LIB_OVERRIDE=ablibs/$v timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.2,1.0,0.01 > gpurun_out/r2c20_sweep_$v.log 2>&1; echo rc=$?
  grep '"m"' gpurun_out/r2c20_sweep_$v.log | head -3
done
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c20_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c20_bench_q.log | head -c 300; echo
