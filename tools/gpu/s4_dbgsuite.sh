mkdir -p gpurun_out
PBNG_LIB=build_variants/libpbng_dbg.so timeout 2400 python -m pytest tests -m gpu -q --durations=3 -k "not host_submission" > gpurun_out/s4_gpu_tests_debug_build.log 2>&1; echo rc=$? >> gpurun_out/s4_gpu_tests_debug_build.log
tail -8 gpurun_out/s4_gpu_tests_debug_build.log
