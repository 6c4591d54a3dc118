mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c47_gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r3c47_gputests.log
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8 --no-prof-leg"
for e in "X=1" "IG_NO_TXT_OVERLAP=1" "X=1" "IG_NO_TXT_OVERLAP=1"; do
env $e timeout 900 python bench.py $A > gpurun_out/r3c47_sd3.log 2>&1; echo "sd3 $e rc=$?"; tail -1 gpurun_out/r3c47_sd3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_step_ms']['median'], d.get('speedup_vs_dense'))"
done
Q="--no-fp8 --no-y --no-lockstep --no-ablation --no-hbm-tier --no-cpu-baseline --no-e2e --no-prof-leg --steps 12 --warmup 4 --dense-steps 0"
for e in "X=1" "IG_NO_TXT_OVERLAP=1" "X=1" "IG_NO_TXT_OVERLAP=1"; do
env $e timeout 900 python bench.py $Q --kv-blocks 24 > gpurun_out/r3c47_flux.log 2>&1; echo "flux $e rc=$?"; tail -1 gpurun_out/r3c47_flux.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done
