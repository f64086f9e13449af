#!/bin/bash
# Round profile refresh on a GPU box (run via gpurun from the repo root):
# ncu launch lists + one --set full capture per config, summarised into
# profiles/ by tools/make_profiles.py, then the bench lines that read them.
# usage: bash tools/refresh_profiles.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out/prof
IFS=';' read -ra SP <<< "${SPECS:-c3 8 4;c5 8 4}"
for spec in "${SP[@]}"; do
  set -- $spec; c=$1; skip=$2; cnt=$3
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/prof/launches_$c.csv python tools/profile_frame.py --config $c --warmup 2 --frames 10 \
    > gpurun_out/prof/launches_$c.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vertex|setup|radix|cm_|tile)" \
    -s $skip -c $cnt -o gpurun_out/prof/full_$c -f python tools/profile_frame.py --config $c --warmup 2 --frames 1 \
    > gpurun_out/prof/full_$c.log 2>&1
  python tools/make_profiles.py ${TAG}_$c gpurun_out/prof/launches_$c.csv gpurun_out/prof/full_$c.ncu-rep $c 16 \
    > gpurun_out/prof/make_$c.log 2>&1
done
for c in ${DRAM_CFGS:-c3}; do
  b=16; [ "$c" = "c6" ] && b=32
  C=$c ARGS="--bin $b" bash tools/frame_dram.sh > /dev/null 2>&1
  cp gpurun_out/prof/frame_dram_$c.csv profiles/frame_dram_${TAG}_$c.csv
  python tools/frame_dram_json.py profiles/frame_dram_${TAG}_$c.csv $c $b
done
for c in ${BENCH_CFGS:-c2 c3 c4 c5}; do
  b=16; [ "$c" = "c6" ] && b=32
  timeout 600 python bench.py --config $c --bin $b > profiles/bench_${TAG}_${c}_b$b.json 2> gpurun_out/prof/bench_$c.err
done
mkdir -p gpurun_out/profiles && cp profiles/* gpurun_out/profiles/
