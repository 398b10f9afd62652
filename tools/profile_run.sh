#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list and full captures of the stage kernel.
#   TAG=r01b tools/profile_run.sh      (outputs in gpurun_out/, summarised into profiles/ by hand)
set -x
TAG=${TAG:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout -s KILL 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu_$TAG.log
timeout -s KILL 300 python __graft_entry__.py > gpurun_out/smoke_$TAG.log 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$TAG.csv \
  python bench.py --steps 2 --warmup 3 --e2e-steps 0 --no-cpu > /dev/null 2>&1
for p in ${PROFILE_ORDERS:-1 5}; do
  ORDERS=$p timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:k_element -s 12 -c 1 \
    -o gpurun_out/prof_${TAG}_p$p python tools/stage_timing.py > gpurun_out/ncu_${TAG}_p$p.log 2>&1
done
# the p=1 limiter on the double-Mach mesh (bench DMR leg)
timeout -s KILL 400 ncu --set full --clock-control none --import-source on -k regex:k_limit -s 6 -c 1 \
  -o gpurun_out/prof_${TAG}_limit python bench.py --orders 1 --no-cpu --e2e-steps 0 --steps 2 --warmup 3 --box 64 \
  > gpurun_out/ncu_${TAG}_limit.log 2>&1
ls -la gpurun_out
