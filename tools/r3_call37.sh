mkdir -p gpurun_out
KB_WARM=0.5 IG_OP_REPEAT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/r3c37_attn128_full python tools/kbench.py --which attn --iters 2 > gpurun_out/r3c37_ncu_a128.log 2>&1; echo rc=$?
KB_WARM=0.5 IG_OP_REPEAT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/r3c37_attn64_full python tools/kbench.py --which attn --iters 2 --dh 64 --heads 10 --L 4096 --qlens 819 --nreq 8 > gpurun_out/r3c37_ncu_a64.log 2>&1; echo rc=$?
