CMD="python bench.py --lines 2000000 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:^compress_tiles -s 1 -c 1 -o gpurun_out/prof_c $CMD > gpurun_out/ncu2.log 2>&1; echo ncu2=$?
