#!/bin/bash
# reference acceptance gate through the adapter under env toggles (bisecting a criterion)
for v in "" "WFK_ASM_LANES_RT=8" "WFK_NO_ASM_SMEM=1" "WFK_NO_HEAVY_DEAL=1"; do
  d=$(mktemp -d)
  (cd $d && env $v OMP_NUM_THREADS=16 timeout 600 $OLDPWD/integration/_build/acceptance_b200 > out.log 2>&1)
  echo "== ${v:-default}: $(grep -c PASS $d/out.log) pass; $(grep 'criterion  2' $d/out.log | cut -c1-160)"
done
