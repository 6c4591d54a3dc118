set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_unet_full.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_unet.py -m gpu -q -x > gpurun_out/r2c14_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c14_pytest.log
timeout 600 python tools/ab_ops.py --op gated --libs ablibs/lib_stage.so,ablibs/lib_nostage.so --shapes "8192,1280,1280;14720,3072,3072;2000,3072,12288;32768,640,640;8192,1280,5120" > gpurun_out/r2c14_gated_ab.txt 2>&1
timeout 600 python tools/ab_ops.py --op attn --libs ablibs/lib_p64_0.so,ablibs/lib_p64_2.so,ablibs/lib_p64_3.so,ablibs/lib_p64_4.so,ablibs/lib_p64_5.so --shapes "64,20,1024,1024,8;64,20,1024,256,8;64,10,4096,4096,8;64,10,4096,820,8;128,24,4608,2355,8" > gpurun_out/r2c14_attn64_ab.txt 2>&1
cat gpurun_out/r2c14_attn64_ab.txt
cat gpurun_out/r2c14_gated_ab.txt
timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.01,0.2,1.0 --out gpurun_out/r2c14_unet_sweep_hbm.json > gpurun_out/r2c14_sweep.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c14_sweep.log | head -3
IG_LIB_OVERRIDE=ablibs/lib_nostage.so timeout 900 python tools/unet_full_sweep.py --tier device --ms 0.2,1.0 > gpurun_out/r2c14_sweep_nostage.log 2>&1; echo rc=$?
grep '"m"' gpurun_out/r2c14_sweep_nostage.log | head -3
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c14_unet_launches_m1.csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
