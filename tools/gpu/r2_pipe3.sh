mkdir -p gpurun_out
python tools/tune_sweep.py --config 3 --iters 10 --reps 5 > gpurun_out/tune_pipe3.jsonl 2>&1
PBNG_SCHEDULE=2 python tools/tune_sweep.py --config 3 --iters 10 --reps 5 >> gpurun_out/tune_pipe3.jsonl 2>&1
python tools/tune_sweep.py --config 3 --dtype f64 --iters 10 --reps 5 >> gpurun_out/tune_pipe3.jsonl 2>&1
PBNG_SCHEDULE=2 python tools/tune_sweep.py --config 3 --dtype f64 --iters 10 --reps 5 >> gpurun_out/tune_pipe3.jsonl 2>&1
