# usage: bash tools/bench_variants.sh "pipe cg"  -- ms/frame of each WFK_PCG variant (2 runs each)
for v in ${1:-pipe cg}; do for i in 1 2; do WFK_PCG=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],3), round(d['e2e']['value'],3), round(d['frame_breakdown_ms']['solve'],3), round(d['roofline']['share_of_frame'],4))"; done; done
