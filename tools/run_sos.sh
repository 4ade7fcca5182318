#!/bin/bash
# Development aid: c2 timings (tools/time_ws.py, AUTO tiling) of library variants copied over the
# in-tree .so one at a time.  usage: tools/run_sos.sh WORKLOAD so1 so2 ...
L=paper_2305_02444_b200/lib/libftblas.so
WL=$1; shift
cp $L /tmp/keep_sos.so
echo "== base"; timeout 200 python tools/time_ws.py $WL auto | grep " ft:"
for so in "$@"; do cp "$so" $L; echo "== $so"; timeout 200 python tools/time_ws.py $WL auto | grep " ft:"; done
cp /tmp/keep_sos.so $L
