# Round-2 final measurements on one B200: bench lines of every config, the reference arm, clocks, and ncu
# captures of the config-3 table-record sweep (fp32 + fp64).  Run from the repo root under gpurun.
mkdir -p gpurun_out
python bench.py > gpurun_out/fb_c3.json 2> gpurun_out/fb_c3.err
for c in 1 2 4 5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/fb_c$c.json 2> gpurun_out/fb_c$c.err; done
python bench.py --config 3 --dtype f64 --no-cpu-baseline > gpurun_out/fb_c3f64.json 2> gpurun_out/fb_c3f64.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/fb_ref_c3.json 2> gpurun_out/fb_ref_c3.err
bash tools/ncu_sweep.sh r2fc3 3
bash tools/ncu_sweep.sh r2fc3d 3 --dtype f64
echo done
