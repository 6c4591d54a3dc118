set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c8_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2c8_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c8_smoke.log 2>&1; echo smoke_rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c8_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
timeout 1800 python bench.py > gpurun_out/r2c8_bench.log 2>&1; echo bench_rc=$?
tail -1 gpurun_out/r2c8_bench.log | head -c 600
timeout 900 python tools/unet_full_sweep.py --tier device --out gpurun_out/r2c8_unet_full_sweep_hbm.json > gpurun_out/r2c8_sweep_hbm.log 2>&1; echo rc=$?
timeout 900 python tools/unet_full_sweep.py --tier host --out gpurun_out/r2c8_unet_full_sweep_host.json > gpurun_out/r2c8_sweep_host.log 2>&1; echo rc=$?
echo done
