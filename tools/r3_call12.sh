mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_unet_full.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/r3c12_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c12_tests.log
for v in gbase gnarrow gbase gnarrow; do
  IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 900 python tools/unet_full_sweep.py --ms 0.2,1.0 --steps 4 --warmup 2 > gpurun_out/r3c12_sweep_$v.log 2>&1; echo $v rc=$?; grep '"m"' gpurun_out/r3c12_sweep_$v.log | cut -c1-200
done
