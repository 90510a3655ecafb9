mkdir -p gpurun_out
python tools/tune_sweep.py --config 4 --iters 10 --reps 5 > gpurun_out/tune_pf.jsonl 2>&1
for v in pf0 pf2 pf8 pf4m4; do echo "== $v" >> gpurun_out/tune_pf.jsonl; PBNG_LIB=build_variants/libpbng_$v.so python tools/tune_sweep.py --config 4 --iters 10 --reps 5 >> gpurun_out/tune_pf.jsonl 2>&1; done
