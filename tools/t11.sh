mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex_slabs.py tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_dist.py -x -q > gpurun_out/t11.log 2>&1; echo "exit $?" >> gpurun_out/t11.log
