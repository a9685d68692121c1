# ncu --set full captures of the two hot kernels at the bench workload
# (C2, 10M lines), after the same command exited 0 without ncu.
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err; rc=$?; echo plain=$rc; cat gpurun_out/plain.json
if [ $rc -eq 0 ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:^compress_tiles -s 3 -c 1 -o gpurun_out/prof_c $CMD > gpurun_out/ncu_c.log 2>&1; echo ncu_c=$?
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:^decompress_tiles -s 3 -c 1 -o gpurun_out/prof_d $CMD > gpurun_out/ncu_d.log 2>&1; echo ncu_d=$?
fi
ls -la gpurun_out
