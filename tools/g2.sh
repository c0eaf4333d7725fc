mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scm.py -m gpu -x -q -k "3d" --timeout 120 > gpurun_out/t3d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d.log
timeout 300 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_parity.py -m gpu -x -q -k "config5 or dist" --timeout 200 > gpurun_out/t3d2.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d2.log
bash tools/ncu_c5.sh
