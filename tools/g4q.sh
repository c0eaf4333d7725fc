mkdir -p gpurun_out
timeout 400 python tools/imex_bench.py 1024 200 > gpurun_out/imex_1024.log 2>&1
timeout 600 python -m pytest tests/test_gpu_elastic.py -m gpu -q --timeout 200 > gpurun_out/t4.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4.log
