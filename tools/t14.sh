mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_iga.py tests/test_gpu_timeint.py tests/test_gpu_imex.py -x -q > gpurun_out/t14.log 2>&1; echo "exit $?" >> gpurun_out/t14.log
timeout 900 python bench.py --config config3 --no-cpu > gpurun_out/b3.json 2> gpurun_out/b3.err
WAVECELL_B200_NO_SHARED_STENCIL=1 timeout 900 python bench.py --config config3 --no-cpu --no-e2e > gpurun_out/b3ns.json 2> gpurun_out/b3ns.err
