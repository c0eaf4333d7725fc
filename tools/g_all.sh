mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
timeout 600 python bench.py --config config4 --steps 3 --warmup 1 --no-cpu > gpurun_out/c4_new.json 2> gpurun_out/c4_new.err
