mkdir -p gpurun_out
Q="--no-fp8 --no-y --no-lockstep --no-ablation --no-hbm-tier --no-cpu-baseline --no-e2e --no-prof-leg --steps 12 --warmup 4 --dense-steps 0"
for k in -1 22 24 26 28 30 -1; do
timeout 900 python bench.py $Q --kv-blocks $k > gpurun_out/r3c46_kv$k.log 2>&1; echo "kv $k rc=$?"; tail -1 gpurun_out/r3c46_kv$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['host_link']['achieved_GBps'], d['config']['impl'][:60], d['clocks']['sm_mhz'])"
done
