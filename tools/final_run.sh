TAG=r01h PROFILE_ORDERS="1 2 5" bash tools/profile_run.sh
timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --same-device --orders 1,3 > gpurun_out/bench_n2_same.json 2> gpurun_out/bench_n2_same.err
timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
