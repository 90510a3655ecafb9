mkdir -p gpurun_out
PBNG_DD_GRAPH=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2s4_dd_transport_launches.csv python tools/dd_transport_profile.py > gpurun_out/s4_ddprof_ncu.log 2>&1; echo rc=$?
python tools/dd_transport_profile.py --summarise gpurun_out/r2s4_dd_transport_launches.csv > gpurun_out/r2s4_dd_transport_summary.md; cat gpurun_out/r2s4_dd_transport_summary.md
(PBNG_PEER_TIMEOUT_MS=5000 timeout 1500 python -m pytest tests -m gpu -x -q -s > gpurun_out/s4_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_gpu_tests.log)
(timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4_smoke.log 2>&1; echo rc=$? >> gpurun_out/s4_smoke.log)
timeout 600 python bench.py > gpurun_out/s4_bench_c3.json 2> gpurun_out/s4_bench_c3.err
tail -3 gpurun_out/s4_gpu_tests.log; grep "us/iteration" gpurun_out/s4_gpu_tests.log; tail -2 gpurun_out/s4_smoke.log; head -c 170 gpurun_out/s4_bench_c3.json
