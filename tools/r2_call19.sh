set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c19_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c19_pytest.log
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c19_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c19_bench_q.log | head -c 300; echo
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c19_unet_sweep_hbm.json > gpurun_out/r2c19_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c19_sweep.log | head -3
