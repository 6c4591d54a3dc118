set -x
mkdir -p gpurun_out
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c11_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c11_bench_q.log | head -c 300; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c11_unet_launches_m02.csv python tools/unet_full_sweep.py --ms 0.2 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c11_unet_launches_m1.csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
timeout 900 python tools/unet_full_sweep.py --tier host --out gpurun_out/r2c11_unet_full_sweep_host.json > gpurun_out/r2c11_sweep_host.log 2>&1; echo rc=$?
