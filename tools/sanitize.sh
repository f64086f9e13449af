# compute-sanitizer over tools/sanitize.py (GPU box): memcheck, racecheck, synccheck
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  echo "== $t"
  timeout 900 ${CS:-/usr/local/cuda/bin/compute-sanitizer} --tool $t --print-limit 20 python tools/sanitize.py 2>&1 | grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error|error|ok$|MISMATCH|done" | head -40
done
