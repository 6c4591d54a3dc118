set -x
timeout 900 python tools/unet_full_sweep.py --tier device --out gpurun_out/r2_unet_full_sweep_hbm.json > gpurun_out/r2c7_sweep_hbm.log 2>&1; echo rc=$?
timeout 900 python tools/unet_full_sweep.py --tier host --out gpurun_out/r2_unet_full_sweep_host.json > gpurun_out/r2c7_sweep_host.log 2>&1; echo rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2c7_unet_launches.csv python tools/unet_full_sweep.py --ms 0.2 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_tc_kernel" -s 200 -c 3 -o gpurun_out/r2c7_conv_full python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 > /dev/null 2>&1; echo rc=$?
