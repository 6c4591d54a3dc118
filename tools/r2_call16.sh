set -x
mkdir -p gpurun_out
KB_WARM=0.5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/r2c16_gated160 python tools/kbench.py --which gated --M 8192 --N 1280 --K 1280 --iters 3 > /dev/null 2>&1; echo rc=$?
IG_GEMM_NO_BN160=1 KB_WARM=0.5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/r2c16_gated256 python tools/kbench.py --which gated --M 8192 --N 1280 --K 1280 --iters 3 > /dev/null 2>&1; echo rc=$?
KB_WARM=0.5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 2 -c 1 -o gpurun_out/r2c16_store160 python tools/kbench.py --which gemm --M 8192 --N 1280 --K 1280 --iters 3 > /dev/null 2>&1; echo rc=$?
for v in p64_0 p64_2 p64_3 p64_4 p64_5; do
  for sh in "--dh 64 --heads 20 --L 1024 --qlens 1024 --nreq 8" "--dh 64 --heads 10 --L 4096 --qlens 4096 --nreq 8" "--dh 64 --heads 10 --L 4096 --qlens 820 --nreq 8"; do
    echo "== $v $sh"
    IG_LIB_OVERRIDE=ablibs/lib_$v.so KB_WARM=0.3 IG_OP_REPEAT=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.max --clock-control none -k regex:attn_tc -s 10 -c 5 --csv python tools/kbench.py --which attn $sh --iters 2 2>/dev/null | grep -E "sm__cycles_elapsed|gpu__time" | awk -F'","' '{gsub(/"/,"",$NF); print $(NF-2), $NF}'
  done
done > gpurun_out/r2c16_attn64_ncu.txt 2>&1
cat gpurun_out/r2c16_attn64_ncu.txt | head -80
