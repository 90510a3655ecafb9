#!/bin/bash
# bash tools/gpu_tune2.sh "<config> <dtype>" <variant>...   (like gpu_tune.sh, with a dtype)
read CFG DT <<< "$1"; shift
mkdir -p gpurun_out
for v in "$@"; do
  if [ "$v" = base ]; then lib=paper_2306_09021_b200/libpbng.so; else lib=build_variants/libpbng_$v.so; fi
  echo -n "$v " >> gpurun_out/tune.jsonl
  PBNG_LIB=$lib timeout 300 python tools/tune_sweep.py --config $CFG --dtype $DT --iters 10 --reps 5 >> gpurun_out/tune.jsonl 2>> gpurun_out/tune.err
done
