mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_imex_slabs.py tests/test_gpu_paper.py tests/test_gpu_tensor.py -m gpu -q --timeout 300 > gpurun_out/t4.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4.log
timeout 600 python tools/imex_bench.py 1024 200 > gpurun_out/imex_1024.log 2>&1
WAVECELL_B200_TRSV_GROUPS=0 timeout 600 python tools/imex_bench.py 1024 200 > gpurun_out/imex_1024_nogroups.log 2>&1
timeout 600 python -m pytest tests/test_gpu_bench_parity.py -m gpu -q -k "config4" --timeout 300 > gpurun_out/t4b.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4b.log
