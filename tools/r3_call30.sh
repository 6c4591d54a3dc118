mkdir -p gpurun_out
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
IG_BENCH_STEP_TRACE=1 timeout 900 python bench.py $A > gpurun_out/r3c30_sd3.log 2> gpurun_out/r3c30_sd3.err; echo sd3 rc=$?; tail -1 gpurun_out/r3c30_sd3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_step_ms'])"
grep "^step" gpurun_out/r3c30_sd3.err | awk '{h=$5; a=$8; if (h+0 > 2 || a+0 > 2) print}' | head -40
