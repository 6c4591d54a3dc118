mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "attention or tiny or flux_small" > gpurun_out/r3c9_tests.log 2>&1; echo rc=$?; tail -2 gpurun_out/r3c9_tests.log
HEADS=24 NOCHECK=1 IG_LIB_OVERRIDE=ablibs/lib_tr_sipp.so timeout 120 python tools/dbg_attn.py 4608 2355,2355,2355,2355,2355,2355,2355,2355 > gpurun_out/r3c9_tr_sipp.txt 2>&1; echo rc=$?
bash tools/ab_cyc.sh gpurun_out/r3c9_cyc.txt ablibs/lib_pp0.so ablibs/lib_sipp.so ablibs/lib_sipp_p8.so ablibs/lib_sipp_p4.so ablibs/lib_sipp_p2.so
