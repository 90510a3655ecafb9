mkdir -p gpurun_out
(timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s4_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_gpu_tests.log)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4_smoke.log 2>&1; echo rc=$? >> gpurun_out/s4_smoke.log)
timeout 600 python bench.py > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err
timeout 600 python bench.py --colouring kuhn4 > gpurun_out/s4_bench_c3_kuhn4.json 2> gpurun_out/s4_bench_c3_kuhn4.err
timeout 600 python bench.py --colouring kuhn4 --dtype f64 --no-cpu-baseline > gpurun_out/s4_bench_c3f64_kuhn4.json 2> gpurun_out/s4_bench_c3f64_kuhn4.err
NCU_DROP_REP=1 timeout 900 bash tools/ncu_sweep.sh r2s4k4 3 --colouring kuhn4 > gpurun_out/s4_ncu.log 2>&1
tail -3 gpurun_out/s4_gpu_tests.log; tail -2 gpurun_out/s4_smoke.log; head -c 300 gpurun_out/s4_bench_c3.json; echo; head -c 300 gpurun_out/s4_bench_c3_kuhn4.json; echo; tail -2 gpurun_out/s4_ncu.log
