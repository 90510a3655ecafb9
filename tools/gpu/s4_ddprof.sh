mkdir -p gpurun_out
PBNG_DD_GRAPH=0 timeout 900 python tools/dd_transport_profile.py > gpurun_out/s4_ddprof_plain.log 2>&1; echo rc=$?
PBNG_DD_GRAPH=0 timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/r2s4_dd_transport_launches.csv python tools/dd_transport_profile.py > gpurun_out/s4_ddprof_ncu.log 2>&1; echo rc=$?
python tools/dd_transport_profile.py --summarise gpurun_out/r2s4_dd_transport_launches.csv
