# round-2 verification: whole GPU suite, smoke, bench lines of every config, reference arm
mkdir -p gpurun_out
PBNG_PARITY_LOG=gpurun_out/parity_full3.jsonl python -m pytest tests -m gpu -q --durations=15 > gpurun_out/pytest_full4.log 2>&1; echo rc=$? >> gpurun_out/pytest_full4.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke4.log 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/bench4_clocks.csv &
SMI=$!
python bench.py > gpurun_out/b4_c3.json 2> gpurun_out/b4_c3.err
for c in 4 2 5 1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/b4_c$c.json 2> gpurun_out/b4_c$c.err; done
python bench.py --config 3 --dtype f64 --no-cpu-baseline > gpurun_out/b4_c3f64.json 2> gpurun_out/b4_c3f64.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/b4_ref.json 2> gpurun_out/b4_ref.err
kill $SMI
