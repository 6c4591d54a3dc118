set -x
mkdir -p gpurun_out
for s in 0 5 9; do
timeout 900 ncu --profile-from-start off --kernel-name-base demangled --set full --clock-control none --import-source on -k regex:"gemm_tc2_kernel<.bool.1" -s $s -c 1 -o gpurun_out/r2c23_conv_s$s python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > gpurun_out/r2c23_conv_s$s.log 2>&1; echo rc=$?
done
ls -la gpurun_out/
