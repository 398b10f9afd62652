mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur vA vB cur vA vB; do
  o=1,2; case $v in cur) o=1,2,3,4,5;; esac
  DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=$o timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
timeout -s KILL 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu_lam.log
