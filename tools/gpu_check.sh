# quick GPU cycle: parity tests, phase profile, then a bench line
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -15 gpurun_out/gpu_tests.log
python tools/phase_profile.py 2000000 2>&1 | tail -12
python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
