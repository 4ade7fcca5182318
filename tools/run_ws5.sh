#!/bin/bash
# ws kernel check (development aid): GPU tests restricted to the ws tiling, timings, phase sums
OUT=gpurun_out/ws5; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "ws" > $OUT/test_ws.log 2>&1; echo "tests rc=$?"; tail -3 $OUT/test_ws.log
for wl in c2_rankk_16384x256 c1_4096_tn c3_16384_sharded; do
  timeout 300 python tools/time_ws.py $wl ws 2>&1 | tail -2
done
cp paper_2305_02444_b200/lib/libftblas.so /tmp/keep.so
for v in ${VARIANTS:-e2p3}; do
  for m in ft noft; do WS_PROF_SO=../var/ws_${v}_FTB_WS_PROF.so timeout 200 python tools/ws_phases.py c2_rankk_16384x256 $m; done
done
cp /tmp/keep.so paper_2305_02444_b200/lib/libftblas.so
[ -n "$ROLES" ] && timeout 600 python tools/ws_roles.py run c2_rankk_16384x256 ws $ROLES 2>&1 | grep median
true
