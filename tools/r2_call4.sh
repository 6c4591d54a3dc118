set -x
python -m pytest tests/test_gpu_pipeline.py -m gpu -x -q > gpurun_out/r2c4_pipeline.log 2>&1; echo rc=$?
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s > gpurun_out/r2c4_full.log 2>&1; echo rc=$?
Q="--no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg"
python bench.py $Q > gpurun_out/r2c4_bench_lane.log 2>&1; echo rc=$?
IG_NO_COPY_THREAD=1 python bench.py $Q > gpurun_out/r2c4_bench_nolane.log 2>&1; echo rc=$?
for v in base max3 st2 st4 max3st2 poly8 poly4 max3st2p8 max3st4p4; do
  for r in 1 2; do
    KB_WARM=0.5 IG_LIB_OVERRIDE=ablibs/lib_$v.so IG_OP_REPEAT=1 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:attn_tc -s 20 -c 10 --csv python tools/kbench.py --which attn --iters 3 2>/dev/null | grep gpu__time_duration | awk -F'","' -v L=$v '{gsub(/"/,"",$NF); print L, $NF}' | sort -k2 -n | awk '{a[NR]=$2; l=$1} END {print l, "median_us", a[int(NR/2)+1], "min_us", a[1], "n", NR}'
  done
done > gpurun_out/r2c4_attn_ab.txt 2>&1
