mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r3c11_gputests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r3c11_gputests.log
timeout 900 python bench.py > gpurun_out/r3c11_bench.log 2>&1; echo bench rc=$?; tail -c 600 gpurun_out/r3c11_bench.log
