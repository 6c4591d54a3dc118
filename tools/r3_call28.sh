mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c28_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c28_gputests.log
timeout 900 python tools/unet_full_sweep.py --ms 0.01,0.2,0.5,1.0 --steps 4 --warmup 2 --out gpurun_out/r3c28_unet_sweep.json > gpurun_out/r3c28_unet_sweep.log 2>&1; echo sweep rc=$?; grep '"m"' gpurun_out/r3c28_unet_sweep.log | head -4 | cut -c1-140
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8"
timeout 900 python bench.py $A > gpurun_out/r3c28_sd3.log 2>&1; echo sd3 rc=$?; tail -1 gpurun_out/r3c28_sd3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d.get('speedup_vs_dense'), d['step_roofline']['frac'], d['clocks'])"
