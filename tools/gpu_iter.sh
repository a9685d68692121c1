# iteration cycle on one B200: parity tests (optional -k filter), one bench
# line, and the compress phase split from the -DZS_PHASES=1 build
set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider ${TESTK:+-k "$TESTK"} > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 20 ${BENCH_ARGS:-} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
ZS_LIB=paper_2404_19391_b200/libzs_phases.so timeout 300 python tools/phase_cx.py 2000000 2>&1 | tail -22
