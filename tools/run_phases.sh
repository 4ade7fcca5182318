#!/bin/bash
# phase sums of the FX persistent kernel vs the FTB_WS_FIXSUM=0 one (development aid)
cp paper_2305_02444_b200/lib/libftblas.so /tmp/keep.so
for so in ${PROFS:-ws_prof_fx.so ws_prof_fx0.so}; do
  for m in ft noft; do echo "== $so"; WS_PROF_SO=$so timeout 200 python tools/ws_phases.py ${WL:-c2_rankk_16384x256} $m; done
done
cp /tmp/keep.so paper_2305_02444_b200/lib/libftblas.so
