#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list and full captures.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt
timeout 1200 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --orders 1,3,5 --e2e-steps 0 --no-cpu > /dev/null 2>&1
for p in ${PROFILE_ORDERS:-1 5}; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_element -s 9 -c 1 \
    -o gpurun_out/prof_p$p python bench.py --steps 1 --warmup 3 --orders $p --e2e-steps 0 --no-cpu > gpurun_out/ncu_p$p.log 2>&1
done
ls -la gpurun_out
