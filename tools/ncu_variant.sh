#!/bin/bash
# ncu --set full of the fused stage kernel for selected orders with a given library build.
mkdir -p gpurun_out
LIBV=${LIBV:-}
for p in ${ORDERS:-1 5}; do
  DGB_LIB=$LIBV ORDERS=$p N=708 timeout 400 ncu --set full --clock-control none --import-source on -k regex:k_element -s 12 -c 1 \
    -o gpurun_out/prof_${TAG:-x}_p$p python tools/stage_timing.py > gpurun_out/ncu_${TAG:-x}_p$p.log 2>&1
done
