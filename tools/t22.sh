mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_elastic.py tests/test_gpu_imex.py tests/test_gpu_timeint.py tests/test_gpu_dist.py -x -q > gpurun_out/t22.log 2>&1; echo "exit $?" >> gpurun_out/t22.log
timeout 300 python tools/step_bench.py config2 1000 3 > gpurun_out/t22_steps.log 2>&1
timeout 400 python tools/imex_bench.py 1024 200 2>&1 | tail -1 >> gpurun_out/t22_steps.log
