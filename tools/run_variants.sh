#!/bin/bash
# GPU session: parity tests on the main build, then stage timing of each variant.
mkdir -p gpurun_out
rm -f gpurun_out/variants.jsonl gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/ -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1
for v in ${VARIANTS:-v1 v2 v3 v4}; do
  DGB_LIB=build/variants/$v/libdg2d_b200.so timeout 240 python tools/stage_timing.py >> gpurun_out/variants.jsonl 2>&1
done
