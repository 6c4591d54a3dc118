mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c20_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c20_gputests.log
timeout 900 python bench.py --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation > gpurun_out/r3c20_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/r3c20_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['step_roofline']['frac'], d['clocks'])"
