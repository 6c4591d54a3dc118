mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -x -q -m gpu -k "gemm or sd3 or tiny or flux_small" > gpurun_out/r3c15_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c15_tests.log
cyc() {
  IG_LIB_OVERRIDE= KB_WARM=0.3 timeout 300 ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:gemm_tc -s 3 -c 2 --csv python tools/kbench.py --iters 3 "$@" 2>/dev/null | grep -E "sm__" | awk -F'","' '{gsub(/"/,"",$NF); gsub(/,/,"",$NF); printf "%s ", $NF}'
  echo
}
for e in "" "IG_GEMM_NO_BN64=1"; do
  echo -n "$e gated 449x1536x6144: "; env $e bash -c "$(declare -f cyc); cyc --which gated --M 449 --N 1536 --K 6144"
  echo -n "$e gated 300x1536x1536: "; env $e bash -c "$(declare -f cyc); cyc --which gated --M 300 --N 1536 --K 1536"
  echo -n "$e gelu 449x6144x1536: "; env $e bash -c "$(declare -f cyc); cyc --which gemm --M 449 --N 6144 --K 1536 --epi 1"
done
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
for e in "X=1" "IG_GEMM_NO_BN64=1" "X=1" "IG_GEMM_NO_BN64=1"; do
  env $e timeout 900 python bench.py $A > gpurun_out/r3c15_sd3_$e.log 2>&1; echo "$e" rc=$?; tail -1 gpurun_out/r3c15_sd3_$e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('speedup_vs_dense'), d['clocks']['sm_mhz'])"
done
