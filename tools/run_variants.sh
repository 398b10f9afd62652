#!/bin/bash
# Stage-kernel timing of tuning builds made by tools/build_variants.sh, interleaved so that
# box-to-box noise cancels:  VARIANTS="base v1" ORDERS=3,4,5 tools/run_variants.sh
mkdir -p gpurun_out
rm -f gpurun_out/variants.jsonl
for v in ${VARIANTS:-base} ${VARIANTS:-base}; do
  DGB_LIB=${VDIR:-build/variants}/$v/libdg2d_b200.so ORDERS=${ORDERS:-1,2,3,4,5} timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
