timeout 400 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout=240 -x > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
bash tools/bench_variants.sh pipe | sed "s/^/L2 /"
for L in 1 4; do WFK_LIBRARY=tools/variants/L$L/libwfk.so bash tools/bench_variants.sh pipe | sed "s/^/L$L /"; done
WFK_PHASE_TIMING=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>&1 >/dev/null | grep "wfk phase" | tail -3
