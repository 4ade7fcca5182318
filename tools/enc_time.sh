#!/bin/bash
# encode_kernel device time (ncu, c1 shape) for each given library build
python tools/prof_c1_lib.py "$1" > /dev/null || exit 1
for l in "$@"; do
  t=$(ncu --metrics gpu__time_duration.sum -k regex:encode --clock-control none --csv python tools/prof_c1_lib.py "$l" 2>/dev/null | grep encode_kernel | tail -1 | awk -F'","' '{print $NF}' | tr -d '"')
  echo "$l encode_ns=$t"
done
