set -x
df -h /dev/shm; free -g | head -2
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s > gpurun_out/r2c3_full.log 2>&1; echo rc=$?
timeout 1200 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "flux_small_batch_end_to_end and 1-1" > gpurun_out/r2c3_racecheck_flux_small.log 2>&1; echo rc=$?
timeout 1500 python bench.py > gpurun_out/r2c3_bench.log 2>&1; echo rc=$?
