mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur out lm6 lm7 cur out lm6 lm7; do
  case $v in cur|out) DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=1,2 timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl;; esac
  DGB_LIB=vlib/$v/libdg2d_b200.so timeout -s KILL 300 python bench.py --orders 1 --no-cpu --e2e-steps 0 --steps 10 --warmup 3 --box 64 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['dmr']['stage_kernel_ms_per_stage'], d['dmr']['limiter_ms_per_stage'])" >> gpurun_out/variants.jsonl
done
DGB_LIB=vlib/out/libdg2d_b200.so timeout -s KILL 900 python -m pytest tests/ -x -q -m gpu 2>&1 | tail -5 > gpurun_out/pytest_gpu_out.log
