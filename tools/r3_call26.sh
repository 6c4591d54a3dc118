mkdir -p gpurun_out
IG_LIB_OVERRIDE=ablibs/lib_smr_p4.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "attention or tiny or flux_small" > gpurun_out/r3c26_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c26_tests.log
bash tools/ab_cyc.sh gpurun_out/r3c26_cyc.txt ablibs/lib_b0.so ablibs/lib_smr.so ablibs/lib_smr_p8.so ablibs/lib_smr_p4.so ablibs/lib_smr_p2.so
