# round-2 session-3 verification: GPU suite, smoke, bench lines of configs 3 and 4, config-4 shard timing
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/s3_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/s3_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3_smoke.log 2>&1; echo rc=$? >> gpurun_out/s3_smoke.log
python bench.py > gpurun_out/s3_bench_c3.json 2> gpurun_out/s3_bench_c3.err
python bench.py --config 4 --no-cpu-baseline > gpurun_out/s3_bench_c4.json 2> gpurun_out/s3_bench_c4.err
timeout 600 python tools/shard_timing.py --n 1 2 4 8 --windows 0 8 > gpurun_out/s3_shard_timing.jsonl 2> gpurun_out/s3_shard.err
