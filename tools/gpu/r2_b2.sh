mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_dd.py tests/test_gpu_dynamics.py tests/test_gpu_contacts.py tests/test_gpu_schedule.py -q -x > gpurun_out/pytest_b2.log 2>&1
echo rc=$? >> gpurun_out/pytest_b2.log
python tools/tune_sweep.py --config 4 --iters 10 --reps 5 > gpurun_out/tune_b2.jsonl 2>&1
for v in m5 m6 m7 m6u4 m1u4 m6u1; do echo "== $v" >> gpurun_out/tune_b2.jsonl; PBNG_LIB=build_variants/libpbng_$v.so python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_b2.jsonl 2>&1; done
