# full GPU test suite + c3 bench line (summary printed)
timeout 1200 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/gpu_tests.log | tail -15
for c in ${CFGS:-c3}; do
  timeout 300 python bench.py --config $c ${BENCH_ARGS:---no-cpu --no-e2e} --steps 30 > gpurun_out/bench_${c}.json 2> gpurun_out/bench_${c}.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}.json'));print('$c', round(d['ms_per_step']*1000,1), [round(x*1000,1) for x in d['ms_p10_p50_p90']], {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'fp', round(d['variants']['freepipe']['ms_per_step']*1000,1))" || tail -3 gpurun_out/bench_${c}.err
done
