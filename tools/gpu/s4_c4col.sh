mkdir -p gpurun_out
timeout 900 python tools/colouring_timing.py --config 4 --reps 3 > gpurun_out/s4_colouring_timing_c4.jsonl 2> gpurun_out/s4_colouring_timing_c4.err
cat gpurun_out/s4_colouring_timing_c4.jsonl; tail -3 gpurun_out/s4_colouring_timing_c4.err
