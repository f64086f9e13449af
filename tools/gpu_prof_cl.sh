mkdir -p gpurun_out/prof
C=${C:-c3}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"${K:-k_setup|k_cl_bins}" -s ${S:-4} -c ${N:-2} -o gpurun_out/prof/cl_$C -f python tools/profile_frame.py --config $C --warmup 2 --frames 1 > gpurun_out/prof/cl_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/cl_$C.ncu-rep
