mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_longlines.py -q -x > gpurun_out/ll_tests.log 2>&1; echo tests=$?
tail -3 gpurun_out/ll_tests.log
ZS_LIB=paper_2404_19391_b200/libzs_checks.so timeout 900 python -m pytest tests/test_gpu_longlines.py -q -x > gpurun_out/ll_tests_c.log 2>&1; echo checks=$?
tail -2 gpurun_out/ll_tests_c.log
timeout 300 python tools/ll_check.py --time-only > gpurun_out/lltime.log 2>&1; echo a=$?
cat gpurun_out/lltime.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ll_ncu.csv python tools/ll_check.py --time-only --size 14000000 > gpurun_out/ll_ncu.log 2>&1; echo ncu=$?
