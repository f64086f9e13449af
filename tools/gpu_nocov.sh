# A/B of the no-coverage compaction (PIKO_NOCOV) after the GPU tests
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -3 gpurun_out/gpu_tests.log
AB="PIKO_NOCOV=1;PIKO_NOCOV=0" CFGS="${CFGS:-c3 c2 c4 c5}" bash tools/gpu_bench_ab.sh
