mkdir -p gpurun_out
PBNG_DD_GRAPH=0 timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_dd.py -x -q -m gpu -k "peer_store_transport_is_bitwise or batched_sample_minor_peer" > gpurun_out/s4_peer_memcheck.log 2>&1; echo rc=$? >> gpurun_out/s4_peer_memcheck.log
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_dd.py -x -q -m gpu -k "peer_store_transport_split" > gpurun_out/s4_peer_memcheck_graph.log 2>&1; echo rc=$? >> gpurun_out/s4_peer_memcheck_graph.log
tail -4 gpurun_out/s4_peer_memcheck.log; tail -4 gpurun_out/s4_peer_memcheck_graph.log
timeout 600 python bench.py > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err
timeout 600 python bench.py --colouring kuhn4 > gpurun_out/s4_bench_c3_kuhn4.json 2> gpurun_out/s4_bench_c3_kuhn4.err
head -c 200 gpurun_out/s4_bench_c3.json
