mkdir -p gpurun_out
python -m pytest tests/test_gpu_schedule.py tests/test_gpu_parity.py -q -x -k "window or batched or config4 or odd" > gpurun_out/pytest_win.log 2>&1; echo rc=$? >> gpurun_out/pytest_win.log
python tools/tune_sweep.py --config 4 --iters 10 --reps 5 > gpurun_out/tune_win.jsonl 2>&1
for w in 1 2 8 16 0; do echo "== window $w" >> gpurun_out/tune_win.jsonl; PBNG_B2_WINDOW=$w python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_win.jsonl 2>&1; done
