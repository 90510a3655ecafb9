mkdir -p gpurun_out
PBNG_LIB=build_variants/libpbng_dbg.so python tools/sanitize_paths.py > gpurun_out/sanitize_dbg2.log 2>&1; echo rc=$? >> gpurun_out/sanitize_dbg2.log
PBNG_LIB=build_variants/libpbng_dbg.so python -m pytest tests/test_gpu_path_records.py tests/test_gpu_dd.py tests/test_gpu_contacts.py -q -x > gpurun_out/pytest_dbg2.log 2>&1; echo rc=$? >> gpurun_out/pytest_dbg2.log
python -m pytest tests -m gpu -q --durations=10 > gpurun_out/pytest_full3.log 2>&1; echo rc=$? >> gpurun_out/pytest_full3.log
