mkdir -p gpurun_out
PBNG_PEER_TIMEOUT_MS=3000 timeout 900 python -m pytest tests/test_gpu_dd.py -x -q -s -m gpu > gpurun_out/s4_dd_tests.log 2>&1; echo rc=$? >> gpurun_out/s4_dd_tests.log
tail -4 gpurun_out/s4_dd_tests.log; grep "us/iteration" gpurun_out/s4_dd_tests.log
PBNG_DD_GRAPH=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2s4_dd_transport_launches.csv python tools/dd_transport_profile.py > gpurun_out/s4_ddprof_ncu.log 2>&1; echo rc=$?
python tools/dd_transport_profile.py --summarise gpurun_out/r2s4_dd_transport_launches.csv
