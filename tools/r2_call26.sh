set -x
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c26_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c26_pytest.log
timeout 900 python tools/unet_full_sweep.py --tier device --out gpurun_out/r2c26_unet_full_sweep_hbm.json > gpurun_out/r2c26_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c26_sweep.log
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c26_unet_launches_m02.csv python tools/unet_full_sweep.py --ms 0.2 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c26_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c26_bench_q.log | head -c 300; echo
