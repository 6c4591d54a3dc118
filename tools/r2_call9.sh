set -x
mkdir -p gpurun_out
timeout 300 python tools/dma_probe.py > gpurun_out/r2c9_dma_probe.json 2> gpurun_out/r2c9_dma_probe.err; echo rc=$?
cat gpurun_out/r2c9_dma_probe.json
Q="--no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 900 python bench.py $Q --copy-mode 1 > gpurun_out/r2c9_bench_cm1.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c9_bench_cm1.log | head -c 300; echo
timeout 900 python bench.py $Q --copy-mode 2 > gpurun_out/r2c9_bench_cm2.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c9_bench_cm2.log | head -c 300; echo
