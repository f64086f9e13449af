python tools/ab.py --prebuilt c3 16 scratch_libs/libpiko_base.so
PIKO_DEFERRED=1 python tools/ab.py --prebuilt c3 16 scratch_libs/libpiko_base.so scratch_libs/libpiko_q1.so
mkdir -p gpurun_out/prof
PIKO_DEFERRED=1 timeout 600 ncu --set full --clock-control none -k regex:"k_shade|k_tile" -s 6 -c 2 -o gpurun_out/prof/defer -f python tools/profile_frame.py --config c3 --warmup 3 --frames 1 > gpurun_out/prof/defer.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/defer.ncu-rep
