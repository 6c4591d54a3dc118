mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "attention or tiny or flux_small" > gpurun_out/r3c7_tests.log 2>&1; echo rc=$?; tail -2 gpurun_out/r3c7_tests.log
HEADS=24 NOCHECK=1 IG_LIB_OVERRIDE=ablibs/lib_tr_wr.so timeout 120 python tools/dbg_attn.py 4608 2355,2355,2355,2355,2355,2355,2355,2355 > gpurun_out/r3c7_tr_wr.txt 2>&1; echo rc=$?
bash tools/ab_cyc.sh gpurun_out/r3c7_cyc.txt ablibs/lib_pp0.so ablibs/lib_wr.so ablibs/lib_wr_p0.so ablibs/lib_wr_p8.so ablibs/lib_wr_p4.so
