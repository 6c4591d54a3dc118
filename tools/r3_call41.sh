mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c41_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c41_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r3c41_bench.log 2>&1; echo bench rc=$?; tail -1 gpurun_out/r3c41_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['step_roofline']['frac'], d['attn_roofline']['frac'], d['roofline']['frac'], d['hbm_tier']['value'], d['clocks'])"
