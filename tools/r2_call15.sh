set -x
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2c15_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2c15_pytest.log
timeout 600 python tools/ab_ops.py --op attn --libs ablibs/lib_p64_0.so,ablibs/lib_p64_2.so,ablibs/lib_p64_3.so,ablibs/lib_p64_4.so,ablibs/lib_p64_5.so --shapes "64,20,1024,1024,8;64,20,1024,256,8;64,10,4096,4096,8;64,10,4096,820,8;128,24,4608,2355,8" > gpurun_out/r2c15_attn64_ab.txt 2>&1
python -c "
import json; d=json.load(open('gpurun_out/r2c15_attn64_ab.txt'))
for sh,v in d.items(): print(sh, {k: v[k]['tflops'] for k in v})"
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c15_unet_sweep_hbm.json > gpurun_out/r2c15_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c15_sweep.log | head -3
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c15_unet_launches_m1.csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
Q="--no-e2e --no-hbm-tier --no-fp8 --no-lockstep --no-ablation --dense-steps 0 --no-cpu-baseline --no-prof-leg --steps 6 --warmup 3"
timeout 1200 python bench.py $Q > gpurun_out/r2c15_bench_q.log 2>&1; echo rc=$?
tail -1 gpurun_out/r2c15_bench_q.log | head -c 300; echo
