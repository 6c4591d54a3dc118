set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r2c5_pytest.log 2>&1; echo rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c5_smoke.log 2>&1; echo rc=$?
Q="--no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --dense-steps 2 --no-cpu-baseline --steps 6 --warmup 3"
IG_BENCH_SHARE_GPU=1 timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 $Q > gpurun_out/r2c5_bench_n2share.log 2>&1; echo rc=$?
timeout 900 python bench.py $Q > gpurun_out/r2c5_bench_n1.log 2>&1; echo rc=$?
