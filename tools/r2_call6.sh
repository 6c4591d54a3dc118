set -x
timeout 1200 python -m pytest tests/test_gpu_unet_full.py -m gpu -x -q > gpurun_out/r2c6_unet_full.log 2>&1; echo rc=$?
tail -30 gpurun_out/r2c6_unet_full.log
