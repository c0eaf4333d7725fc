mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_dist.py tests/test_gpu_bench_parity.py -m gpu -x -q -k "not 3d and not config5 and not config4" --timeout 300 > gpurun_out/t2d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t2d.log
timeout 300 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/c2_new.json 2> gpurun_out/c2_new.err
WAVECELL_B200_NO_DIRECT2D=1 timeout 300 python bench.py --config config2 --steps 5 --warmup 3 --no-cpu --no-e2e --no-secondary > gpurun_out/c2_old.json 2> gpurun_out/c2_old.err
