mkdir -p gpurun_out
(timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s4_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_gpu_tests.log)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4_smoke.log 2>&1; echo rc=$? >> gpurun_out/s4_smoke.log)
timeout 600 python bench.py > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/s4_bench_c4.json 2> gpurun_out/s4_bench_c4.err
timeout 600 python bench.py --config 5 --no-cpu-baseline > gpurun_out/s4_bench_c5.json 2> gpurun_out/s4_bench_c5.err
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/s4_bench_c2.json 2> gpurun_out/s4_bench_c2.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/s4_ref_c3.json 2> gpurun_out/s4_ref_c3.err
tail -3 gpurun_out/s4_gpu_tests.log; tail -2 gpurun_out/s4_smoke.log; for f in c3 c4 c5 c2; do head -c 160 gpurun_out/s4_bench_$f.json; echo; done; head -c 300 gpurun_out/s4_ref_c3.json
