mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_timeint.py -x -q > gpurun_out/t7.log 2>&1; echo "exit $?" >> gpurun_out/t7.log
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:trsv|ela2d<\(int\)5, \(int\)0>' -c 12 --log-file gpurun_out/launches_trsv_fix.csv python tools/imex_bench.py 1024 3 > gpurun_out/ncu_trsv_fix.log 2>&1
timeout 300 python tools/step_bench.py config2 500 3 > gpurun_out/l2.log 2>&1
WAVECELL_B200_L2_PERSIST=1 timeout 300 python tools/step_bench.py config2 500 3 >> gpurun_out/l2.log 2>&1
timeout 900 python bench.py --config config4 > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
