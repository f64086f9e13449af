# A/B of prebuilt compile-time variants (tools/ab.py --build-only LIBS first), piko_draw frames
L=${LIBS:-$(ls scratch_libs/*.so)}
for c in ${CFGS:-"c3 16" "c2 16" "c4 16" "c5 16"}; do AB_DRAW=${AB_DRAW:-draw} timeout 600 python tools/ab.py --prebuilt $c $L; done
