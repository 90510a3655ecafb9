mkdir -p gpurun_out
python -m pytest tests/test_gpu_dd.py tests/test_gpu_dynamics.py tests/test_gpu_parity.py -q -x -s > gpurun_out/pytest_dd.log 2>&1
echo rc=$? >> gpurun_out/pytest_dd.log
