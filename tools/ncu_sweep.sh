#!/bin/bash
# ncu evidence for the sweep kernel (run on a GPU box via gpurun): plain run, launch list, full capture.
# usage: bash tools/ncu_sweep.sh <tag> [bench args...]
TAG=${1:-r1}; shift
ARGS=${@:-"--steps 1 --warmup 3 --no-cpu-baseline --no-e2e"}
CMD="python bench.py $ARGS"
mkdir -p gpurun_out
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 450 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 9 -c 2 -o gpurun_out/${TAG}_sweep $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo "exit $?"
