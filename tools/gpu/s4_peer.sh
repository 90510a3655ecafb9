mkdir -p gpurun_out
PBNG_PEER_TIMEOUT_MS=3000 timeout 900 python -m pytest tests/test_gpu_dd.py -x -q -s -m gpu > gpurun_out/s4_dd_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_dd_tests.log
tail -15 gpurun_out/s4_dd_tests.log
