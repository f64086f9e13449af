mkdir -p gpurun_out/prof
for c in c3 c5; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vertex|setup|radix|cm_|tile)" \
    -s 8 -c 4 -o gpurun_out/prof/full_$c -f python tools/profile_frame.py --config $c --warmup 2 --frames 1 \
    > gpurun_out/prof/full_$c.log 2>&1
done
AB="X=0;PIKO_CM_TC_LOG2=11;PIKO_CM_TC_LOG2=13" CFGS="c3" bash tools/gpu_bench_ab.sh
AB="X=0;PIKO_CM_TC_LOG2=15;PIKO_CM_TC_LOG2=17" CFGS="c5" bash tools/gpu_bench_ab.sh
