mkdir -p gpurun_out
IG_LIB_OVERRIDE=ablibs/lib_lnw1.so timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/r3c19_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c19_tests.log
A="--steps 3 --warmup 3 --no-e2e --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --no-prof-leg --dense-steps 3"
for v in lnw0 lnw1; do
  IG_LIB_OVERRIDE=ablibs/lib_$v.so IG_BENCH_PROFILE_STEP=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r3c19_launches_$v.csv python bench.py $A > gpurun_out/r3c19_ncu_$v.log 2>&1; echo $v rc=$?
  python tools/launch_summary.py gpurun_out/r3c19_launches_$v.csv | grep -E "ln_mod|launches,"
done
