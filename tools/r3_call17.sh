mkdir -p gpurun_out
cyc() {
  lib=$1; shift
  IG_LIB_OVERRIDE=$lib KB_WARM=0.3 timeout 300 ncu --metrics sm__cycles_elapsed.max --clock-control none -k regex:gemm_tc -s 3 -c 2 --csv python tools/kbench.py --iters 3 "$@" 2>/dev/null | grep -E "sm__" | awk -F'","' '{gsub(/"/,"",$NF); gsub(/,/,"",$NF); printf "%s ", $NF}'
  echo
}
for lib in ablibs/lib_pf0.so ablibs/lib_pf16.so ablibs/lib_pf32.so ablibs/lib_pf64.so; do
  echo -n "$lib gated449x1536x6144: "; cyc $lib --which gated --M 449 --N 1536 --K 6144
  echo -n "$lib gated300x1536x1536: "; cyc $lib --which gated --M 300 --N 1536 --K 1536
  echo -n "$lib gelu449x6144x1536: "; cyc $lib --which gemm --M 449 --N 6144 --K 1536 --epi 1
  echo -n "$lib gated2048x1280x5120: "; cyc $lib --which gated --M 2048 --N 1280 --K 5120
done > gpurun_out/r3c17_cyc.txt 2>&1
cat gpurun_out/r3c17_cyc.txt
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
for v in pf0 pf32 pf0 pf32; do
  IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 900 python bench.py $A > gpurun_out/r3c17_sd3_$v.log 2>&1; echo "$v" rc=$?; tail -1 gpurun_out/r3c17_sd3_$v.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('speedup_vs_dense'), d.get('dense_images_per_s'), d['clocks'])"
done
