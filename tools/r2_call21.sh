set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 2400 python bench.py > gpurun_out/r2c21_bench_final.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/r2c21_bench_final.log | head -c 400; echo
timeout 1200 python bench.py --model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 > gpurun_out/r2c21_bench_sd3.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c21_bench_sd3.log | head -c 300; echo
timeout 900 python tools/unet_full_sweep.py --tier device --out gpurun_out/r2c21_unet_full_sweep_hbm.json > gpurun_out/r2c21_sweep_hbm.log 2>&1; echo rc=$?
timeout 900 python tools/unet_full_sweep.py --tier host --out gpurun_out/r2c21_unet_full_sweep_host.json > gpurun_out/r2c21_sweep_host.log 2>&1; echo rc=$?
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 3 --warmup 3 --no-y"
IG_BENCH_PROFILE_STEP=1 timeout 1200 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r2c21_flux_step_launches.csv python bench.py $Q > gpurun_out/r2c21_ncu_step.log 2>&1; echo rc=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c21_unet_launches_m02.csv python tools/unet_full_sweep.py --ms 0.2 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
