mkdir -p gpurun_out
for c in 2 5; do
timeout 900 python tools/colouring_timing.py --config $c --reps 3 >> gpurun_out/s4_colouring_timing_c25.jsonl 2>> gpurun_out/s4_colouring_timing_c25.err
done
cat gpurun_out/s4_colouring_timing_c25.jsonl; tail -3 gpurun_out/s4_colouring_timing_c25.err
