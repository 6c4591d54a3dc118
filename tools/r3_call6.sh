mkdir -p gpurun_out
HEADS=24 NOCHECK=1 IG_LIB_OVERRIDE=ablibs/lib_tr_tp.so timeout 120 python tools/dbg_attn.py 4608 2355,2355,2355,2355,2355,2355,2355,2355 > gpurun_out/r3c6_tr_tp.txt 2>&1; echo rc=$?
bash tools/ab_cyc.sh gpurun_out/r3c6_cyc.txt ablibs/lib_pp0.so ablibs/lib_tp.so ablibs/lib_tp_p0.so ablibs/lib_tp_p8.so ablibs/lib_tp_p4.so ablibs/lib_tp_p2.so
