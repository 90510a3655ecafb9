mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_given_colouring.py -x -q -m gpu > gpurun_out/s4_colour_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_colour_tests.log
tail -6 gpurun_out/s4_colour_tests.log
