set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/r2c10_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c10_pytest.log
timeout 300 python tools/dma_probe.py > gpurun_out/r2c10_dma_probe.json 2> gpurun_out/r2c10_dma_probe.err; echo rc=$?
cat gpurun_out/r2c10_dma_probe.json
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c10_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c10_bench_q.log | head -c 400; echo
KB_WARM=0.5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 3 -c 1 -o gpurun_out/r2c10_gemm_full python tools/kbench.py --which gemm --M 14720 --N 21504 --K 3072 --iters 2 > gpurun_out/r2c10_ncu_gemm.log 2>&1; echo rc=$?
KB_WARM=0.5 IG_OP_REPEAT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/r2c10_attn_full python tools/kbench.py --which attn --iters 2 > gpurun_out/r2c10_ncu_attn.log 2>&1; echo rc=$?
timeout 300 python tools/kbench.py --which gemm,attn > gpurun_out/r2c10_kbench.json 2>&1; echo rc=$?
cat gpurun_out/r2c10_kbench.json
