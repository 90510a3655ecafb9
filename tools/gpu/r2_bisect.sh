mkdir -p gpurun_out
PBNG_LIB=build_variants/libpbng_head.so python tools/gpu/dbg_relayout.py gpurun_out/dbg_head.json > gpurun_out/dbg_head.log 2>&1
python tools/gpu/dbg_relayout.py gpurun_out/dbg_cur.json > gpurun_out/dbg_cur.log 2>&1
