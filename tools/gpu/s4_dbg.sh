mkdir -p gpurun_out
PBNG_LIB=build_variants/libpbng_dbg.so timeout 900 python tools/sanitize_paths.py > gpurun_out/s4_debug_sanitize_paths.log 2>&1; echo rc=$? >> gpurun_out/s4_debug_sanitize_paths.log
PBNG_LIB=build_variants/libpbng_dbg.so PBNG_PEER_TIMEOUT_MS=3000 timeout 900 python -m pytest tests/test_gpu_dd.py -x -q -m gpu -k "peer" >> gpurun_out/s4_debug_sanitize_paths.log 2>&1; echo rc=$? >> gpurun_out/s4_debug_sanitize_paths.log
tail -8 gpurun_out/s4_debug_sanitize_paths.log
NCU_DROP_REP=1 timeout 900 bash tools/ncu_sweep.sh r2s4c3 3 > gpurun_out/s4_ncu_c3.log 2>&1
tail -2 gpurun_out/s4_ncu_c3.log
