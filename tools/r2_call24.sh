set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_unet_full.py -m gpu -q -x > gpurun_out/r2c24_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2c24_pytest.log
for v in lib_conv2d.so lib_conv4d.so; do
  IG_LIB_OVERRIDE=ablibs/$v timeout 900 python tools/unet_full_sweep.py --tier device --ms 1.0,0.2,0.01 > gpurun_out/r2c24_sweep_$v.log 2>&1; echo rc=$?
  grep '"m"' gpurun_out/r2c24_sweep_$v.log | head -3
done
for s in 0 5 9; do
timeout 900 ncu --profile-from-start off --kernel-name-base demangled --metrics gpu__time_duration.sum,sm__cycles_elapsed.max,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:"gemm_tc2_kernel<.bool.1" -s $s -c 1 --csv python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile 2>/dev/null | grep -E "gpu__time|cycles_elapsed|tensor" | awk -F'","' '{gsub(/"/,"",$NF); print $(NF-2), $NF}'
done
