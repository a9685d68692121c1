# one ncu --set full capture of compress_cx at the bench workload (after the
# plain tests/bench exited 0), summaries into gpurun_out/
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:^compress_cx -s 3 -c 1 \
  -o gpurun_out/full_compress -f $CMD > gpurun_out/ncu_c.log 2>&1; echo ncu_compress=$?
