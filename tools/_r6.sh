mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "async" 2>&1 | tail -5 > gpurun_out/pytest_gpu_async.log
timeout -s KILL 600 python bench.py --no-cpu --dmr-nx 0 --steps 5 --warmup 3 > gpurun_out/bench_async.json 2> gpurun_out/bench_async.err
