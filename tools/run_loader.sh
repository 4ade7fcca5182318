#!/bin/bash
# VERDICT r1 item 8 experiment (development aid): FT 128 x 128 kernel with and without the
# loader-side encoding sums (tools/variant_build.py loader_encode), c1 and c3
L=paper_2305_02444_b200/lib/libftblas.so
cp $L /tmp/keep.so
for wl in c1_4096_tn c3_16384_sharded; do echo "== base $wl"; timeout 300 python tools/time_ws.py $wl full | tail -2; done
cp tools/var/loader_encode.so $L
for wl in c1_4096_tn c3_16384_sharded; do echo "== loader_encode $wl"; timeout 300 python tools/time_ws.py $wl full | tail -2; done
cp /tmp/keep.so $L
