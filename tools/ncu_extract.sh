#!/bin/bash
# Development aid: export the parts of an ncu report that profiles/ keeps, then delete the report
# (gpurun brings back at most 64 MiB).  usage: ncu_extract.sh <report-without-ext>
r=$1
ncu -i $r.ncu-rep --page raw --csv > $r.raw.csv 2>/dev/null
ncu -i $r.ncu-rep --page source --csv --print-source sass > $r.src.csv 2>/dev/null
gzip -f $r.src.csv
rm -f $r.ncu-rep
