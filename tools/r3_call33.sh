mkdir -p gpurun_out
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
for r in 1 2 3; do
IG_GRAPH_TRACE=1 IG_BENCH_STEP_TRACE=1 timeout 900 python bench.py $A > gpurun_out/r3c33_sd3_$r.log 2> gpurun_out/r3c33_sd3_$r.err; echo "run $r" rc=$?; tail -1 gpurun_out/r3c33_sd3_$r.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_step_ms'])"
grep -E "IG_GRAPH_TRACE: (graphs|evicted)" gpurun_out/r3c33_sd3_$r.err | tail -12
grep "^step" gpurun_out/r3c33_sd3_$r.err | awk '{if ($5+0 > 20) print}'
done
