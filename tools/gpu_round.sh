# round evidence: parity tests, smoke, full default bench line, then the ncu
# launch list of the same bench command (only if it exited 0)
set -u
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -6 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo bench=$rc; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_bench.log 2>&1; echo ncu=$?
fi
