mkdir -p gpurun_out/c2cache
python tools/parity_variants.py gpurun_out/c2cache > gpurun_out/c2acc.jsonl 2> gpurun_out/c2acc.err
for v in pf64 n8 j6 n8j6; do PBNG_LIB=build_variants/libpbng_$v.so python tools/parity_variants.py gpurun_out/c2cache >> gpurun_out/c2acc.jsonl 2>> gpurun_out/c2acc.err; done
rm -rf gpurun_out/c2cache
