set -x
Q="--no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --dense-steps 2 --no-cpu-baseline --steps 4 --warmup 3"
IG_BENCH_SHARE_GPU=1 timeout 1800 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 $Q > gpurun_out/r2c27_bench_n2share.log 2>&1; echo rc=$?
tail -2 gpurun_out/r2c27_bench_n2share.log | head -c 1500; echo
