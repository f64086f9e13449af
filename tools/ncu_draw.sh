mkdir -p gpurun_out/prof
for spec in "c3 8 4" "c5 8 4"; do
  set -- $spec; c=$1; skip=$2; cnt=$3
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_" --csv \
    --log-file gpurun_out/prof/launches_$c.csv python tools/profile_frame.py --config $c --warmup 2 --frames 10 \
    > gpurun_out/prof/launches_$c.log 2>&1
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(vertex|setup|radix|cm_|tile)" \
    -s $skip -c $cnt -o gpurun_out/prof/full_$c -f python tools/profile_frame.py --config $c --warmup 2 --frames 1 \
    > gpurun_out/prof/full_$c.log 2>&1
  python tools/make_profiles.py r2_$c gpurun_out/prof/launches_$c.csv gpurun_out/prof/full_$c.ncu-rep $c 16 > gpurun_out/prof/make_$c.log 2>&1
done
mkdir -p gpurun_out/profiles && cp profiles/launches_r2_* profiles/ncu_full_r2_* profiles/traffic_c* gpurun_out/profiles/
cat profiles/launches_r2_c3.txt profiles/ncu_full_r2_c3.txt
