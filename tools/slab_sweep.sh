#!/bin/bash
# Slab-partitioned CG sweep on one B200 (run through gpurun from the repo
# root): frame-1 solve of configs[3] / configs[4], fused (no slabs) and
# S = 1, 2, 4, 8 virtual ranks; one JSON line per run into
# gpurun_out/slab_sweep.jsonl (energy_final_hex shows the runs are bit-identical).
mkdir -p gpurun_out
: > gpurun_out/slab_sweep.jsonl
for c in 3 4; do
  for s in 0 1 2 4 8; do
    timeout 300 python bench.py --solve-config $c --steps 10 --warmup 3 --slabs $s 2>/dev/null >> gpurun_out/slab_sweep.jsonl
  done
done
python - <<'PY'
import json
for line in open("gpurun_out/slab_sweep.jsonl"):
    d = json.loads(line)
    print(d["config"]["lattice"][0], d["config"]["parallelism"][:110], round(d["value"], 2), d["energy_final_hex"])
PY
