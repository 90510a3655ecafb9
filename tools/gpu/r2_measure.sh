set -x
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/alu_peaks tools/alu_peaks.cu
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/alu_clocks.csv &
SMI=$!
./tools/alu_peaks > gpurun_out/alu_peaks.json 2> gpurun_out/alu_peaks.err
kill $SMI
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
for c in 2 4 5 1; do python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_c$c.json 2> gpurun_out/bench_c$c.err; done
python bench.py --config 3 --dtype f64 --no-cpu-baseline > gpurun_out/bench_c3f64.json 2> gpurun_out/bench_c3f64.err
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/ref_c3.json 2> gpurun_out/ref_c3.err
PBNG_PARITY_LOG=gpurun_out/parity_c2seeds.jsonl python -m pytest tests/test_gpu_parity_full.py -q -k config2 > gpurun_out/pytest_c2seeds.log 2>&1
python tools/flop_count.py > gpurun_out/flops_plain.log 2>&1 && \
ncu --profile-from-start off --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/flops.csv python tools/flop_count.py > gpurun_out/flops_ncu.log 2>&1
echo done
