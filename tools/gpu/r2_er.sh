mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py tests/test_gpu_contacts.py tests/test_gpu_dynamics.py tests/test_gpu_dd.py -q -x > gpurun_out/pytest_er.log 2>&1; echo rc=$? >> gpurun_out/pytest_er.log
python bench.py --config 4 --no-cpu-baseline > gpurun_out/b3_c4.json 2> gpurun_out/b3_c4.err
python tools/contact_timing.py --n 32 48 --steps 12 --iters 40 > gpurun_out/contact_timing.jsonl 2> gpurun_out/contact_timing.err
