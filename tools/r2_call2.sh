set -x
python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -m gpu -x -q -k "pipeline or dedupe or staggered or poison or dropped or corrupt or mask_build or dump or tile" > gpurun_out/r2c2_pytest.log 2>&1; echo rc=$?
python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -k "teacher_forced_block" > gpurun_out/r2c2_full_default.log 2>&1; echo rc=$?
IG_PRECISE_GELU=1 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -s -k "teacher_forced_block" > gpurun_out/r2c2_full_precise.log 2>&1; echo rc=$?
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiny_config" > gpurun_out/r2c2_racecheck.log 2>&1; echo rc=$?
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tiny_config" > gpurun_out/r2c2_synccheck.log 2>&1; echo rc=$?
