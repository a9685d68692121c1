# ncu --set full of one kernel (regex $KREGEX) at the bench workload
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${BENCH_ARGS:-}"
timeout 600 $CMD > gpurun_out/plain.json 2> gpurun_out/plain.err; rc=$?; echo plain=$rc; cat gpurun_out/plain.json
[ $rc -eq 0 ] && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 3 -c 1 -o gpurun_out/${NAME:-prof} $CMD > gpurun_out/ncu.log 2>&1; echo ncu=$?
