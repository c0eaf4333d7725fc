mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_elastic.py tests/test_gpu_dist.py -m gpu -x -q --timeout 300 > gpurun_out/t2d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t2d.log
timeout 300 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/c2_new.json 2> gpurun_out/c2_new.err
