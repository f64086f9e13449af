timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gpu_tests.log
tail -2 gpurun_out/gpu_tests.log
L="scratch_libs/libpiko_base.so scratch_libs/libpiko_tiny32.so scratch_libs/libpiko_t32tpt1.so scratch_libs/libpiko_t32tpt1m6.so"
for c in "c3 16" "c2 16" "c4 16" "c5 16"; do AB_DRAW=draw timeout 600 python tools/ab.py --prebuilt $c $L; done
