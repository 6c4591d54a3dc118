set -x
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "attention or tiny or flux_small" > gpurun_out/r3c1_tests.log 2>&1; echo rc=$?; tail -3 gpurun_out/r3c1_tests.log
L=ablibs/lib_pp0.so,ablibs/lib_pp1.so,ablibs/lib_pp1_p8.so,ablibs/lib_pp1_p4.so
timeout 600 python tools/ab_ops.py --libs $L --op attn --rounds 7 --shapes "128,24,4608,2355,8;128,24,4608,1331,8;64,10,4096,819,8;64,20,1024,1024,8;64,10,4096,4096,8" > gpurun_out/r3c1_ab.json 2>&1; echo rc=$?
cat gpurun_out/r3c1_ab.json
