# A/B of prebuilt compile-time variants (tools/ab.py --build-only LIBS first), piko_draw frames
# usage: CFGS="c3:16 c2:16" bash tools/gpu_abrun.sh
L=${LIBS:-$(ls scratch_libs/*.so)}
for cb in ${CFGS:-c3:16 c2:16 c4:16 c5:16}; do
  AB_DRAW=${AB_DRAW:-draw} timeout 600 python tools/ab.py --prebuilt ${cb%%:*} ${cb##*:} $L
done
