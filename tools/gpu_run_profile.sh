set -x
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench=$?; cat gpurun_out/bench.json
CMD="python bench.py --lines 2000000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1; echo ncu1=$?
ncu --set full --clock-control none --import-source on -k regex:compress_tiles -s 3 -c 1 -o gpurun_out/prof_c $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
ncu --set full --clock-control none --import-source on -k regex:decompress_tiles -s 3 -c 1 -o gpurun_out/prof_d $CMD > gpurun_out/ncu3.log 2>&1; echo ncu3=$?
ls -la gpurun_out
