CMD="python tools/phase_profile_d.py 1000000"
$CMD > gpurun_out/plain_d.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:decompress_tiles_bp -s 2 -c 1 -o gpurun_out/prof_d $CMD > gpurun_out/ncu_d.log 2>&1; echo ncu=$?
