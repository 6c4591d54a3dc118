mkdir -p gpurun_out
Q="--no-fp8 --no-y --no-lockstep --no-ablation --no-hbm-tier --no-cpu-baseline --no-e2e --no-prof-leg --steps 12 --warmup 4 --dense-steps 0 --kv-blocks 24"
for dp in 8 12 16 8 12 16; do
timeout 900 python bench.py $Q --depth $dp > gpurun_out/r3c48_d$dp.log 2>&1; echo "depth $dp rc=$?"; tail -1 gpurun_out/r3c48_d$dp.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['host_link']['achieved_GBps'], d['clocks']['sm_mhz'])"
done
