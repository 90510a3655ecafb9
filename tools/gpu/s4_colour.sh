mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_given_colouring.py -x -q -m gpu > gpurun_out/s4_colour_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_colour_tests.log
tail -4 gpurun_out/s4_colour_tests.log
timeout 600 python tools/colouring_timing.py --dtype f32 > gpurun_out/s4_colouring_timing.jsonl 2> gpurun_out/s4_colouring_timing.err
timeout 600 python tools/colouring_timing.py --dtype f64 >> gpurun_out/s4_colouring_timing.jsonl 2>> gpurun_out/s4_colouring_timing.err
cat gpurun_out/s4_colouring_timing.jsonl; tail -3 gpurun_out/s4_colouring_timing.err
