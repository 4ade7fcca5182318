#!/bin/bash
# encode_kernel device time (ncu, c1 shape) for each given library build
TB=${TB:-T}
python tools/prof_c1_lib.py "$1" $TB > /dev/null || exit 1
for l in "$@"; do
  t=$(ncu --metrics gpu__time_duration.sum -k regex:encode --clock-control none --csv python tools/prof_c1_lib.py "$l" $TB 2>/dev/null | grep encode_kernel | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')
  echo "$l encode_ns=$t"
done
