set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x > gpurun_out/r2c18_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c18_pytest.log
cyc() {
  lib=$1; k=$2; shift 2
  IG_LIB_OVERRIDE=ablibs/$lib KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:$k -s 6 -c 4 --csv python tools/kbench.py "$@" --iters 3 2>/dev/null | grep -E "sm__cycles_elapsed" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'
  echo
}
for v in lib_gbase.so lib_gred.so; do
  for sh in "8192 1280 1280" "32768 640 640" "8192 1280 5120" "14720 3072 3072" "14720 3072 15360" "3000 3072 3072"; do set -- $sh; echo -n "$v gated $sh: "; cyc $v gemm_tc2 --which gated --M $1 --N $2 --K $3; done
done > gpurun_out/r2c18_gated_cyc.txt 2>&1
cat gpurun_out/r2c18_gated_cyc.txt
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c18_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c18_bench_q.log | head -c 300; echo
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c18_unet_sweep_hbm.json > gpurun_out/r2c18_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c18_sweep.log | head -3
