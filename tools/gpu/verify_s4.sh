mkdir -p gpurun_out
(timeout 1500 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s4_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_gpu_tests.log)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4_smoke.log 2>&1; echo rc=$? >> gpurun_out/s4_smoke.log)
timeout 600 python bench.py > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err
tail -3 gpurun_out/s4_gpu_tests.log; tail -2 gpurun_out/s4_smoke.log; head -c 600 gpurun_out/s4_bench_c3.json
