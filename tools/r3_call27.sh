mkdir -p gpurun_out
bash tools/ab_cyc.sh gpurun_out/r3c27_cyc.txt ablibs/lib_b0.so ablibs/lib_smr.so ablibs/lib_smr_c.so ablibs/lib_smr_c3.so
