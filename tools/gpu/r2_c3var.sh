mkdir -p gpurun_out
python tools/tune_sweep.py --config 3 --iters 10 --reps 5 > gpurun_out/tune_c3var.jsonl 2>&1
for v in m8 m10 u3 u4 m8u3 pf8; do echo "== $v" >> gpurun_out/tune_c3var.jsonl; PBNG_LIB=build_variants/libpbng_$v.so python tools/tune_sweep.py --config 3 --iters 10 --reps 5 >> gpurun_out/tune_c3var.jsonl 2>&1; done
