mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "attention or tiny or flux_small" > gpurun_out/r3c5_tests.log 2>&1; echo rc=$?; tail -3 gpurun_out/r3c5_tests.log
for v in tp tp_p4; do
HEADS=24 NOCHECK=1 IG_LIB_OVERRIDE=ablibs/lib_tr_$v.so timeout 120 python tools/dbg_attn.py 4608 2355,2355,2355,2355,2355,2355,2355,2355 > gpurun_out/r3c5_tr_$v.txt 2>&1; echo rc=$?
done
L=ablibs/lib_pp0.so,ablibs/lib_tp.so,ablibs/lib_tp_p0.so,ablibs/lib_tp_p8.so,ablibs/lib_tp_p4.so,ablibs/lib_tp_p2.so
timeout 900 python tools/ab_ops.py --libs $L --op attn --rounds 7 --shapes "128,24,4608,2355,8;128,24,4608,1331,8;64,10,4096,819,8;64,20,1024,1024,8;64,10,4096,4096,8" > gpurun_out/r3c5_ab.json 2>&1; echo rc=$?
python - <<'P'
import json; d=json.load(open("gpurun_out/r3c5_ab.json"))
for sh,v in d.items(): print(sh, {k[4:-3]: x["tflops"] for k,x in v.items()})
P
