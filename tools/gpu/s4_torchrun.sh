mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/s4_torchrun_w1.json 2> gpurun_out/s4_torchrun_w1.err; echo rc=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --config 5 --steps 3 --warmup 3 --no-cpu-baseline --halo peer > gpurun_out/s4_torchrun_w1_c5.json 2> gpurun_out/s4_torchrun_w1_c5.err; echo rc=$?
head -c 200 gpurun_out/s4_torchrun_w1.json; echo; tail -3 gpurun_out/s4_torchrun_w1.err; head -c 200 gpurun_out/s4_torchrun_w1_c5.json; echo; tail -3 gpurun_out/s4_torchrun_w1_c5.err
