#!/bin/bash
# fixed-point epilogue verification check (development aid): timings of the shipped lib and of the
# variants in tools/var/ (VARS, e.g. "fx0 r30"), then (unless NOTEST) the GPU suite on the shipped lib
OUT=gpurun_out/fx; mkdir -p $OUT
LIB=paper_2305_02444_b200/lib/libftblas.so
cp $LIB /tmp/new.so
for wl in ${WLS:-c2_rankk_16384x256 c1_4096_tn}; do
  echo "== new $wl"; timeout 300 python tools/time_ws.py $wl ws 2>&1 | tail -2
done
for v in $VARS; do
  cp tools/var/$v.so $LIB
  for wl in ${WLS:-c2_rankk_16384x256 c1_4096_tn}; do
    echo "== $v $wl"; timeout 300 python tools/time_ws.py $wl ws 2>&1 | tail -2
  done
done
cp /tmp/new.so $LIB
if [ -z "$NOTEST" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q ${PYK:+-k "$PYK"} > $OUT/test.log 2>&1; echo "tests rc=$?"; tail -15 $OUT/test.log
fi
true
