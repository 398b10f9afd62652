mkdir -p gpurun_out; rm -f gpurun_out/variants.jsonl
for v in cur r1 r3 u3 mb mmaU t3 cur r1 r3 u3 mb mmaU t3; do
  o=1,2; case $v in cur) o=1,2,3,4,5;; mmaU) o=5;; t3) o=3;; esac
  DGB_LIB=vlib/$v/libdg2d_b200.so ORDERS=$o timeout -s KILL 200 python tools/stage_timing.py >> gpurun_out/variants.jsonl
done
