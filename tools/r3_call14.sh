mkdir -p gpurun_out
A="--model sd3_medium --max-batch 1 --tier device --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 6 --warmup 3 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --no-prof-leg --dense-steps 3"
IG_BENCH_PROFILE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r3c14_sd3_launches.csv python bench.py $A > gpurun_out/r3c14_ncu.log 2>&1; echo rc=$?
