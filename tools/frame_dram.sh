# usage (GPU box): C=c3 bash tools/frame_dram.sh
C=${C:-c3}
mkdir -p gpurun_out/prof
timeout 600 ncu --replay-mode range --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
  --csv --log-file gpurun_out/prof/frame_dram_$C.csv python tools/frame_dram.py --config $C ${ARGS:-} > gpurun_out/prof/frame_dram_$C.log 2>&1
tail -12 gpurun_out/prof/frame_dram_$C.csv
