#!/bin/bash
# One GPU-box session: bench line, then (plain run && ncu) launch list of a short bench command,
# and one ncu --set full capture of the first FT GEMM launch.  Usage: tools/gpu_bench_profile.sh TAG [WORKLOAD]
TAG=${1:-run}; WL=${2:-c3_16384_sharded}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 600 python bench.py --workload $WL > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
tail -1 $OUT/bench.json
CMD="python bench.py --workload $WL --steps 1 --warmup 3 --skip-cpu --skip-e2e"
timeout 300 $CMD > $OUT/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv $CMD > $OUT/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
if [ "${FULL:-1}" = 1 ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -c 1 -o $OUT/ft_full $CMD > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
ls -la $OUT
