mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_dist.py -x -q > gpurun_out/t9.log 2>&1; echo "exit $?" >> gpurun_out/t9.log
timeout 300 python tools/step_bench.py config5 20 2 > gpurun_out/s5b.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:k_cut_pre|k_scm3d<\(int\)3, \(int\)0>|zcol|zline' -c 12 --log-file gpurun_out/launches_c5step.csv python tools/step_bench.py config5 4 1 > gpurun_out/ncu_c5step.log 2>&1
