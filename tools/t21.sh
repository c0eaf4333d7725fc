mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_iga.py tests/test_gpu_timeint.py -x -q > gpurun_out/t21.log 2>&1; echo "exit $?" >> gpurun_out/t21.log
timeout 900 python bench.py --config config3 --no-cpu --no-e2e > gpurun_out/b3w.json 2> gpurun_out/b3w.err
