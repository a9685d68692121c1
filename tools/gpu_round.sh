# Round evidence on one B200: parity tests, smoke, the default bench line,
# the reference arm, the C5 (1B-line) bench line, the ncu launch list of the
# bench command, and `ncu --set full` captures of the hot kernels at the bench
# workload (each ncu pass only after the plain command exited 0).
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo build failed; exit 1; }
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; rc=$?; echo bench=$rc; cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref=$?; cat gpurun_out/bench_ref.json; tail -3 gpurun_out/bench_ref.err
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err; echo c5=$?
if [ $rc -eq 0 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-check \
    > gpurun_out/ncu_bench.log 2>&1; echo ncu_launches=$?
  CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-check"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:^compress_cx -s 3 -c 1 \
    -o gpurun_out/full_compress -f $CMD > gpurun_out/ncu_c.log 2>&1; echo ncu_compress=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^fx_(count|emit)" -s 6 -c 2 \
    -o gpurun_out/full_decompress -f $CMD > gpurun_out/ncu_d.log 2>&1; echo ncu_decompress=$?
fi
timeout 900 python tools/ll_check.py > gpurun_out/ll_check.log 2>&1; echo ll=$?; tail -8 gpurun_out/ll_check.log
timeout 1500 python tools/configs.py > gpurun_out/configs.json 2> gpurun_out/configs.err; echo configs=$?
