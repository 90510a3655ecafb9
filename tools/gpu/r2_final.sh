# Round-2 final measurements on one B200 (two gpurun calls: gpurun_out/ must stay under 64 MiB per call).
#   bash tools/gpu/r2_final.sh a   -> the GPU suite, smoke, bench lines of every config, the reference arm,
#                                    ncu capture of the config-3 table-record sweep (fp32)
#   bash tools/gpu/r2_final.sh b   -> ncu captures of the config-3 fp64 sweep and the config-4 batched sweep
mkdir -p gpurun_out
if [ "$1" = a ]; then
python -m pytest tests -m gpu -q --durations=8 > gpurun_out/final_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/final_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo rc=$? >> gpurun_out/final_smoke.log
python bench.py > gpurun_out/fb_c3.json 2> gpurun_out/fb_c3.err
for c in 1 2 4 5; do python bench.py --config $c --no-cpu-baseline > gpurun_out/fb_c$c.json 2> gpurun_out/fb_c$c.err; done
python bench.py --config 3 --dtype f64 --no-cpu-baseline > gpurun_out/fb_c3f64.json 2> gpurun_out/fb_c3f64.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/fb_ref_c3.json 2> gpurun_out/fb_ref_c3.err
bash tools/ncu_sweep.sh r2fc3 3
else
NCU_DROP_REP=1 bash tools/ncu_sweep.sh r2fc3d 3 --dtype f64
NCU_DROP_REP=1 bash tools/ncu_sweep.sh r2fc4 4
fi
echo done
