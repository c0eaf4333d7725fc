mkdir -p gpurun_out
timeout 300 python bench.py --config config3 --steps 5 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/c3_new.json 2> gpurun_out/c3_new.err
timeout 900 python -m pytest tests/test_gpu_iga.py tests/test_gpu_timeint.py -m gpu -x -q --timeout 300 > gpurun_out/t3.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3.log
