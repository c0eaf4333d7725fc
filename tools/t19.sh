mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_imex_slabs.py -x -q > gpurun_out/t19.log 2>&1; echo "exit $?" >> gpurun_out/t19.log
timeout 400 python tools/imex_bench.py 1024 200 2>&1 | tail -1 >> gpurun_out/t19b.log
