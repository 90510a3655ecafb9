#!/bin/bash
# ncu evidence for the sweep kernel (run on a GPU box via gpurun): plain run, launch list, full capture of
# one whole iteration (8 colour launches, skipping the first iteration).
# usage: bash tools/ncu_sweep.sh <tag> <config> [extra bench args]
TAG=${1:-r1}; CFG=${2:-3}; shift 2
CMD="python bench.py --config $CFG --steps 1 --warmup 3 --no-cpu-baseline --no-e2e $*"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep -s 8 -c 8 -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
rc=$?
# raw page as CSV next to the report; NCU_DROP_REP=1 deletes the report (gpurun copies back <= 64 MiB)
ncu -i gpurun_out/${TAG}_sweep.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
[ "$NCU_DROP_REP" = 1 ] && rm -f gpurun_out/${TAG}_sweep.ncu-rep
echo "exit $rc"
