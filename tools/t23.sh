mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_imex_slabs.py tests/test_gpu_timeint.py -x -q > gpurun_out/t23.log 2>&1; echo "exit $?" >> gpurun_out/t23.log
timeout 400 python tools/imex_bench.py 1024 200 2>&1 | tail -1 >> gpurun_out/t23b.log
WAVECELL_B200_NO_IMEX_OVERLAP=1 timeout 400 python tools/imex_bench.py 1024 200 2>&1 | tail -1 >> gpurun_out/t23b.log
