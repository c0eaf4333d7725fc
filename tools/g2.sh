mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scm.py -m gpu -x -q -k "3d" --timeout 120 > gpurun_out/t3d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d.log
timeout 300 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
timeout 600 python -m pytest tests/test_gpu_dist.py tests/test_gpu_bench_parity.py -m gpu -x -q -k "config5 or dist" --timeout 200 > gpurun_out/t3d2.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d2.log
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_cut_pre' -s 320 -c 1 -f -o gpurun_out/cut_pre python bench.py --config config5 --nt 6 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_cut.log 2>&1
