mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unet.py tests/test_gpu_pipeline.py -x -q -m gpu -k "graph or tiny or flux_small" > gpurun_out/r3c40_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c40_tests.log
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
timeout 900 python bench.py $A > gpurun_out/r3c40_sd3.log 2>&1; echo sd3 rc=$?; tail -1 gpurun_out/r3c40_sd3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_step_ms'])"
timeout 900 python tools/unet_full_sweep.py --ms 0.2 --steps 4 --warmup 2 > gpurun_out/r3c40_unet.log 2>&1; echo unet rc=$?; grep '"m"' gpurun_out/r3c40_unet.log | head -1 | cut -c1-120
