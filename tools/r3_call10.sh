mkdir -p gpurun_out
bash tools/ab_cyc.sh gpurun_out/r3c10_cyc.txt ablibs/lib_pp0.so ablibs/lib_sp.so ablibs/lib_pp1.so ablibs/lib_pp1_p8.so
