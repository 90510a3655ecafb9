# warm-cache ncu captures (--cache-control none) of the config-3 colour sweep and the config-4 batched sweep:
# L2-slice (LTS) and L1 throughput, hit rates and stall reasons at steady state (raw CSV exported on the box)
mkdir -p gpurun_out
C3="python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
C4="python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
ncu --set full --cache-control none --clock-control none --import-source on -k regex:sweep_kernel -s 16 -c 8 -o gpurun_out/s3c3w $C3 > gpurun_out/s3c3w.log 2>&1
ncu -i gpurun_out/s3c3w.ncu-rep --page raw --csv > gpurun_out/s3c3w_raw.csv 2>/dev/null
ncu --set full --cache-control none --clock-control none -k regex:sweep_batched2 -s 16 -c 8 -o gpurun_out/s3c4w $C4 > gpurun_out/s3c4w.log 2>&1
ncu -i gpurun_out/s3c4w.ncu-rep --page raw --csv > gpurun_out/s3c4w_raw.csv 2>/dev/null
ls -la gpurun_out/
