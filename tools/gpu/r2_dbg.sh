mkdir -p gpurun_out
PBNG_TIMING=1 python -m pytest tests/test_gpu_contacts.py -q -s -k colliding > gpurun_out/pytest_dbg2.log 2>&1; echo rc=$? >> gpurun_out/pytest_dbg2.log
