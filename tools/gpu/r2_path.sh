mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x --deselect tests/test_gpu_parity_full.py > gpurun_out/pytest_path.log 2>&1
echo rc=$? >> gpurun_out/pytest_path.log
for c in 4 3; do python tools/tune_sweep.py --config $c --iters 10 --reps 5 >> gpurun_out/tune_path.jsonl 2>&1; PBNG_PATH=0 python tools/tune_sweep.py --config $c --iters 10 --reps 5 >> gpurun_out/tune_path.jsonl 2>&1; done
python tools/tune_sweep.py --config 3 --dtype f64 --iters 10 --reps 5 >> gpurun_out/tune_path.jsonl 2>&1
PBNG_PATH=0 python tools/tune_sweep.py --config 3 --dtype f64 --iters 10 --reps 5 >> gpurun_out/tune_path.jsonl 2>&1
