mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur r1m5 r1m6 m5 cur r1m5 r1m6 m5; do
  DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=1 timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
