#!/bin/bash
# ws warp-role experiment (development aid): timings of every variant, phase sums of the PROF builds
OUT=gpurun_out/roles; mkdir -p $OUT
cp paper_2305_02444_b200/lib/libftblas.so /tmp/libftblas.keep
timeout 300 python tools/time_ws.py c2_rankk_16384x256 pair > $OUT/pair_c2.txt 2>&1
for wl in c2_rankk_16384x256 c1_4096_tn c3_16384_sharded; do
  timeout 900 python tools/ws_roles.py run $wl ws 0:3 2:3 3:0 3:2 > $OUT/roles_$wl.txt 2>&1
done
for v in e0p3 e3p2 e3p0; do
  for m in ft noft; do
    WS_PROF_SO=../var/ws_${v}_FTB_WS_PROF.so timeout 300 python tools/ws_phases.py c2_rankk_16384x256 $m > $OUT/ph_${v}_$m.txt 2>&1
  done
done
cp /tmp/libftblas.keep paper_2305_02444_b200/lib/libftblas.so
