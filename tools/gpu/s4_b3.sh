mkdir -p gpurun_out
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4_bench_c3_b.json 2> gpurun_out/s4_bench_c3_b.err; echo rc=$?
timeout 600 python bench.py --config 4 --colouring kuhn4 --no-cpu-baseline > gpurun_out/s4_bench_c4_kuhn4.json 2> gpurun_out/s4_bench_c4_kuhn4.err; echo rc=$?
timeout 600 python bench.py --config 5 --colouring kuhn4 --no-cpu-baseline > gpurun_out/s4_bench_c5_kuhn4.json 2> gpurun_out/s4_bench_c5_kuhn4.err; echo rc=$?
for f in c3_b c4_kuhn4 c5_kuhn4; do head -c 170 gpurun_out/s4_bench_$f.json; echo; tail -2 gpurun_out/s4_bench_$f.err; done
