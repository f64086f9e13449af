# A/B of env knobs on the GPU box: parity tests, then bench lines per config
# usage: AB="PIKO_CM=0;PIKO_CM=1" CFGS="c3 c2" bash tools/gpu_ab.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
grep -E "passed|failed|^FAILED|^ERROR" gpurun_out/gpu_tests.log | tail -12
IFS=';' read -ra VARS <<< "${AB:-X=0}"
for c in ${CFGS:-c3 c2 c4}; do for v in "${VARS[@]}"; do
  env $v timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps ${STEPS:-30} > gpurun_out/bench_${c}.json 2> gpurun_out/bench_${c}.err
  python -c "import json;d=json.load(open('gpurun_out/bench_${c}.json'));print('$c $v', round(d['ms_per_step']*1000,1), [round(x*1000,1) for x in d['ms_p10_p50_p90']], {k:round(v*1000,1) for k,v in d['kernel_ms'].items()}, 'fp', round(d['variants']['freepipe']['ms_per_step']*1000,1))" || tail -3 gpurun_out/bench_${c}.err
done; done
