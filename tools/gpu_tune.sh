#!/bin/bash
# Time sweep variants on the GPU box: bash tools/gpu_tune.sh "<configs>" <variant> [<variant> ...]
# variant "base" = paper_2306_09021_b200/libpbng.so, otherwise build_variants/libpbng_<variant>.so
CFGS=$1; shift
mkdir -p gpurun_out
for v in "$@"; do
  for c in $CFGS; do
    if [ "$v" = base ]; then lib=paper_2306_09021_b200/libpbng.so; else lib=build_variants/libpbng_$v.so; fi
    echo -n "$v " >> gpurun_out/tune.jsonl
    PBNG_LIB=$lib timeout 300 python tools/tune_sweep.py --config $c --iters 10 --reps 5 >> gpurun_out/tune.jsonl 2>> gpurun_out/tune.err
  done
done
