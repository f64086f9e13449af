set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
for c in c3 c2 c4 c5; do timeout 300 python bench.py --config $c --no-cpu --no-e2e --steps 30 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; done
tail -2 gpurun_out/gpu_tests.log
cat gpurun_out/bench_c3.json
