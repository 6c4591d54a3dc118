set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_smoke_launches.csv python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
KB_WARM=0.3 ncu --set full --clock-control none --import-source on -k regex:gemm_tc2 -s 3 -c 1 -o gpurun_out/r2_gemm_full python tools/kbench.py --which gemm --M 14720 --N 21504 --K 3072 --iters 2 > gpurun_out/r2_ncu_gemm.log 2>&1
KB_WARM=0.3 IG_OP_REPEAT=1 ncu --set full --clock-control none --import-source on -k regex:attn_tc -s 3 -c 1 -o gpurun_out/r2_attn_full python tools/kbench.py --which attn --iters 2 > gpurun_out/r2_ncu_attn.log 2>&1
python tools/kbench.py --which gemm,attn > gpurun_out/r2_kbench.json 2>&1
echo done
