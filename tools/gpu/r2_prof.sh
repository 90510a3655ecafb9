mkdir -p gpurun_out
bash tools/ncu_sweep.sh r2c3 3
bash tools/ncu_sweep.sh r2c4f 4
python tools/flop_count.py > gpurun_out/flops_plain2.log 2>&1 && \
ncu --profile-from-start off --metrics smsp__sass_thread_inst_executed_op_ffma_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul_pred_on.sum,smsp__sass_thread_inst_executed_op_ffma2_pred_on.sum,smsp__sass_thread_inst_executed_op_fadd2_pred_on.sum,smsp__sass_thread_inst_executed_op_fmul2_pred_on.sum,smsp__sass_thread_inst_executed_op_dfma_pred_on.sum,smsp__sass_thread_inst_executed_op_dadd_pred_on.sum,smsp__sass_thread_inst_executed_op_dmul_pred_on.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/flops2.csv python tools/flop_count.py > gpurun_out/flops_ncu2.log 2>&1
