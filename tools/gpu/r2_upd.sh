mkdir -p gpurun_out
python -m pytest tests/test_gpu_contacts.py tests/test_gpu_dynamics.py tests/test_gpu_dd.py tests/test_gpu_parity.py tests/test_gpu_schedule.py -q -x > gpurun_out/pytest_upd.log 2>&1; echo rc=$? >> gpurun_out/pytest_upd.log
PBNG_TIMING=1 python tools/contact_timing.py --n 32 48 --steps 12 --iters 40 > gpurun_out/contact_timing2.jsonl 2> gpurun_out/contact_timing2.err
