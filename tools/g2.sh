mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scm.py tests/test_gpu_iga.py -m gpu -x -q -k "3d or stencil" --timeout 120 > gpurun_out/t3d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d.log
timeout 300 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
N=/usr/local/cuda/bin/ncu
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:k_cut_pre' -s 320 -c 5 --log-file gpurun_out/launches_cut.csv python bench.py --config config5 --nt 6 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_cut.log 2>&1
