mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur cur; do
  DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=3 timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
timeout -s KILL 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu_half.log
