mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c18_gputests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c18_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r3c18_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/r3c18_smoke.log
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r3c18_ref.log 2>&1; echo ref rc=$?; tail -c 400 gpurun_out/r3c18_ref.log
IG_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 4 --warmup 3 --no-cpu-baseline --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation > gpurun_out/r3c18_n2.log 2>&1; echo n2 rc=$?; tail -c 600 gpurun_out/r3c18_n2.log
