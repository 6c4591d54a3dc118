mkdir -p gpurun_out
rm -f gpurun_out/r3c23_tl.csv
IG_PROFILE_DUMP=$PWD/gpurun_out/r3c23_tl.csv timeout 900 python bench.py --steps 4 --warmup 3 --no-hbm-tier --no-fp8 --no-y --no-lockstep --no-ablation --no-cpu-baseline --no-e2e > gpurun_out/r3c23_bench.log 2>&1; echo rc=$?
wc -l gpurun_out/r3c23_tl.csv
python tools/tl_analyze.py gpurun_out/r3c23_tl.csv | tail -4
python tools/tl_svg.py gpurun_out/r3c23_tl.csv gpurun_out/r3c23_tl.svg
