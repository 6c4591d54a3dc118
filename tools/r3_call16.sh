mkdir -p gpurun_out
KB_WARM=0.3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:gemm_tc -s 3 -c 1 -o gpurun_out/r3c16_small_gated python tools/kbench.py --iters 3 --which gated --M 449 --N 1536 --K 6144 > gpurun_out/r3c16.log 2>&1; echo rc=$?
