set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_unet_full.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/r2c12_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c12_pytest.log
for r in 1 2 3; do for v in split nosplit; do echo -n "$v "; KB_WARM=0.5 IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 300 python tools/kbench.py --which attn; done; done > gpurun_out/r2c12_attn_ab.txt 2>&1
cat gpurun_out/r2c12_attn_ab.txt
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c12_unet_sweep_hbm.json > gpurun_out/r2c12_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c12_sweep.log | head -5
IG_GEMM_NO_BN160=1 timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,1.0 > gpurun_out/r2c12_sweep_no160.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c12_sweep_no160.log | head -3
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c12_unet_launches_m1.csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c12_unet_launches_m02.csv python tools/unet_full_sweep.py --ms 0.2 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
