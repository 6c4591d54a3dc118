set -x
mkdir -p gpurun_out
A2="--which attn --dh 64 --heads 20 --L 1024 --qlens 1024 --nreq 8"
A2m="--which attn --dh 64 --heads 20 --L 1024 --qlens 256 --nreq 8"
A1="--which attn --dh 64 --heads 10 --L 4096 --qlens 4096 --nreq 8"
A1m="--which attn --dh 64 --heads 10 --L 4096 --qlens 820 --nreq 8"
SD3="--which attn --dh 64 --heads 24 --L 1178 --qlens 154,307 --nreq 1"
for r in 1 2; do for v in p64_0 p64_2 p64_3 p64_4 p64_5; do
  for a in A2 A2m A1 A1m SD3; do eval args=\$$a; echo -n "$v $a "; KB_WARM=0.3 IG_LIB_OVERRIDE=ablibs/lib_$v.so timeout 120 python tools/kbench.py $args; done
done; done > gpurun_out/r2c13_attn64_ab.txt 2>&1
cat gpurun_out/r2c13_attn64_ab.txt
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm_tc2_kernel" -s 5 -c 3 -o gpurun_out/r2c13_unet_gemm_full python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
timeout 900 ncu --profile-from-start off --set full --clock-control none --import-source on -k regex:"gemm_tc2_kernel<1" -s 2 -c 2 -o gpurun_out/r2c13_unet_conv_full python tools/unet_full_sweep.py --ms 1.0 --steps 1 --warmup 1 --profile > /dev/null 2>&1; echo rc=$?
