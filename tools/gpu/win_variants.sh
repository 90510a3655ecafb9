mkdir -p gpurun_out
for v in wold wls wls2 wls4; do
  PBNG_LIB=build_variants/libpbng_$v.so timeout 600 python tools/shard_timing.py --n 1 2 4 8 --windows 0 8 16 2>>gpurun_out/win.err | sed "s/^/$v /" >> gpurun_out/win.jsonl
done
for v in wls wls2 wls4; do
  PBNG_LIB=build_variants/libpbng_$v.so timeout 600 python -m pytest tests -m gpu -q -x -k "window" >> gpurun_out/win_tests.log 2>&1; echo "$v rc=$?" >> gpurun_out/win_tests.log
done
