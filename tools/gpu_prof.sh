# c3 per-CTA timeline + ncu --set full (all kernels of one frame, source-level)
mkdir -p gpurun_out/prof
C=${C:-c3}
timeout 300 python tools/cm_timeline.py $C > gpurun_out/prof/timeline_$C.txt 2>&1
tail -40 gpurun_out/prof/timeline_$C.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${K:-k_}" -s ${S:-10} -c ${N:-6} -o gpurun_out/prof/full_$C -f python tools/profile_frame.py --config $C --warmup 2 --frames 1 > gpurun_out/prof/full_$C.log 2>&1
python tools/ncu_summary.py gpurun_out/prof/full_$C.ncu-rep
