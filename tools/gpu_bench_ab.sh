# bench lines (full JSON kept) for env variants: AB="X=0;PIKO_SEPARATE_VS=1" CFGS="c3" bash tools/gpu_bench_ab.sh
IFS=';' read -ra VARS <<< "${AB:-X=0}"
for c in ${CFGS:-c3}; do for v in "${VARS[@]}"; do
  tag=$(echo "$v" | tr '=;' '__')
  env $v timeout 600 python bench.py --config $c ${BENCH_ARGS:---no-e2e} --steps ${STEPS:-30} > gpurun_out/bench_${c}_${tag}.json 2> gpurun_out/bench_${c}_${tag}.err
  python - "$c" "$v" "gpurun_out/bench_${c}_${tag}.json" <<'PY' || tail -5 gpurun_out/bench_${c}_${tag}.err
import json, sys
c, v, f = sys.argv[1:4]
d = json.load(open(f))
vr = d.get("variants", {})
print(c, v, round(d["ms_per_step"] * 1000, 1), [round(x * 1000, 1) for x in d["ms_p10_p50_p90"]],
      {k: round(x * 1000, 1) for k, x in d["kernel_ms"].items() if x > 0.003},
      {k: round(x["ms_per_step"] * 1000, 1) for k, x in vr.items()},
      "parity", d.get("parity", {}).get("ok"), "cpu1", round(d.get("cpu_baseline", {}).get("value", 0), 2),
      "cpuN", d.get("cpu_baseline", {}).get("all_cores", {}).get("value"), "roof", d["roofline"]["kernel"],
      round(d["roofline"]["frac"], 3))
PY
done; done
