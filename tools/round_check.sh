#!/bin/bash
# Round-end evidence on one B200 (run from the repo root through gpurun):
# GPU test suite, smoke, the default bench line and the reference arm.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_final.log 2>&1; tail -3 gpurun_out/gpu_tests_final.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_final.log 2>&1; tail -2 gpurun_out/smoke_final.log
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -c 600 gpurun_out/bench_final.json
python bench.py --impl reference > gpurun_out/reference_arm_final.json 2> gpurun_out/reference_arm_final.err
tail -c 400 gpurun_out/reference_arm_final.json
