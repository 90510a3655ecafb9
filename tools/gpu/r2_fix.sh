mkdir -p gpurun_out
python -m pytest tests/test_gpu_path_records.py tests/test_gpu_schedule.py tests/test_gpu_parity.py tests/test_gpu_dd.py -q > gpurun_out/pytest_fix.log 2>&1; echo rc=$? >> gpurun_out/pytest_fix.log
python bench.py --config 4 --no-cpu-baseline > gpurun_out/b5_c4.json 2> gpurun_out/b5_c4.err
python tools/shard_timing.py --n 8 4 --windows 0 8 > gpurun_out/shard2.jsonl 2>&1
