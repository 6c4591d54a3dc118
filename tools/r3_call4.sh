mkdir -p gpurun_out
for v in p0 sp p8 p4 p2; do
HEADS=24 NOCHECK=1 IG_LIB_OVERRIDE=ablibs/lib_tr_$v.so timeout 120 python tools/dbg_attn.py 4608 2355,2355,2355,2355,2355,2355,2355,2355 > gpurun_out/r3c4_tr_$v.txt 2>&1; echo rc=$?
done
