mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur m1 m3 m5 cur m1 m3 m5; do
  DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=1,2,3,4,5 timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
