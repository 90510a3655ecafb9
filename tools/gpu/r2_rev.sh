mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py -q -x -k "batched or config4 or odd" > gpurun_out/pytest_rev.log 2>&1; echo rc=$? >> gpurun_out/pytest_rev.log
python tools/tune_sweep.py --config 4 --iters 10 --reps 5 > gpurun_out/tune_rev.jsonl 2>&1
for v in m4 m5; do echo "== $v" >> gpurun_out/tune_rev.jsonl; PBNG_LIB=build_variants/libpbng_$v.so python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_rev.jsonl 2>&1; done
