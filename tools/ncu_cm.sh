mkdir -p gpurun_out/prof
C=${C:-c3}
timeout 600 ncu --set full --import-source on --clock-control none --cache-control ${CC:-all} -k regex:"${K:-k_cm|k_setup}" -s ${S:-6} -c ${N:-3} -o gpurun_out/prof/full_$C -f python tools/profile_frame.py --config $C --warmup 2 --frames 1 > gpurun_out/prof/full_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/full_$C.ncu-rep
