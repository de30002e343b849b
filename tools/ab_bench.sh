#!/bin/bash
# A/B of two libwfk builds on one box (run through gpurun): alternating bench
# runs with the in-tree library and WFK_LIBRARY=$1.
for i in 1 2 3; do
  for lib in "" "$1"; do
    WFK_LIBRARY=$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-current}', round(d['value'],3), round(d['e2e']['value'],3))"
  done
done
