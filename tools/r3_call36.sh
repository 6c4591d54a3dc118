mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c36_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c36_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r3c36_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/r3c36_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['step_roofline']['frac'], d['attn_roofline'], d['roofline']['frac'], d['clocks'])"
A="--model sd3_medium --max-batch 1 --tier device --graphs --mask-kind blob --mask-lo 0.1 --mask-hi 0.5 --steps 56 --warmup 8 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --dense-steps 8"
timeout 900 python bench.py $A > gpurun_out/r3c36_sd3.log 2>&1; echo sd3 rc=$?; tail -1 gpurun_out/r3c36_sd3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['per_step_ms'], d.get('speedup_vs_dense'), d['step_roofline']['frac'])"
