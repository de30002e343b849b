#!/bin/bash
# the reference acceptance gate through the adapter, repeated (flakiness check)
for i in $(seq 1 ${1:-4}); do
  d=$(mktemp -d)
  (cd $d && env $2 OMP_NUM_THREADS=16 timeout 600 $OLDPWD/integration/_build/acceptance_b200 > out.log 2>&1)
  echo "== run $i ${2}: $(grep -c PASS $d/out.log) pass; $(grep 'criterion  2' $d/out.log | cut -c60-200)"
done
