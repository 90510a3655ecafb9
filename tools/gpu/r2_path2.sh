mkdir -p gpurun_out
python -m pytest tests/test_gpu_path_records.py -q > gpurun_out/pytest_path2.log 2>&1; echo rc=$? >> gpurun_out/pytest_path2.log
PBNG_LIB=build_variants/libpbng_dbg.so python -m pytest tests/test_gpu_path_records.py tests/test_gpu_dd.py tests/test_gpu_contacts.py tests/test_gpu_schedule.py -q -x > gpurun_out/pytest_dbg2.log 2>&1; echo rc=$? >> gpurun_out/pytest_dbg2.log
