mkdir -p gpurun_out
IG_COPY_STREAMS=2 timeout 1200 python -m pytest tests/test_gpu_pipeline.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/r3c38_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r3c38_tests.log
for v in 1 2; do
IG_COPY_STREAMS=$v timeout 900 python bench.py --no-fp8 --no-lockstep --no-ablation --no-cpu-baseline > gpurun_out/r3c38_bench_$v.log 2>&1; echo "streams $v" rc=$?
tail -1 gpurun_out/r3c38_bench_$v.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); c=d['cache_forms_host_tier']
print(d['value'], d['ms_per_step'], d['host_link'], 'kv', c['kv_bf16_planned (north-star form)']['value'], c['kv_bf16_planned (north-star form)']['host_link_GBps'], 'hbm', d['hbm_tier']['value'], d['config']['impl'], d['clocks']['sm_mhz'])"
done
