mkdir -p gpurun_out
python -m pytest tests/test_gpu_schedule.py -q -x > gpurun_out/pytest_sched.log 2>&1; echo rc=$? >> gpurun_out/pytest_sched.log
python tools/tune_sweep.py --config 4 --iters 10 --reps 5 > gpurun_out/tune_b2p.jsonl 2>&1
PBNG_PATH=0 python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_b2p.jsonl 2>&1
for v in m4 m5 m4u1 m5u1 m6u1 m1; do echo "== $v" >> gpurun_out/tune_b2p.jsonl; PBNG_LIB=build_variants/libpbng_$v.so python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_b2p.jsonl 2>&1; done
