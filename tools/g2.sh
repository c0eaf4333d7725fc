mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_paper.py tests/test_gpu_dist.py tests/test_gpu_bench_parity.py -m gpu -x -q -k "3d or config5 or dist or criterion or paper" --timeout 300 > gpurun_out/t3d.log 2>&1; echo "pytest exit $?" >> gpurun_out/t3d.log
timeout 300 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu --no-e2e > gpurun_out/c5_new.json 2> gpurun_out/c5_new.err
N=/usr/local/cuda/bin/ncu
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:trsv|k_c_|_rows|k_rc_|ela2d<.*5,.*0>|k_imex|k_state' -s 60 -c 300 --log-file gpurun_out/launches_c4.csv python tools/imex_bench.py 1024 40 > gpurun_out/ncu_c4_list.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_trsv_ring' -s 6 -c 1 -f -o gpurun_out/trsv_ring python tools/imex_bench.py 1024 6 > gpurun_out/ncu_c4_trsv.log 2>&1
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:scm3d|cut_pre' -s 700 -c 40 --log-file gpurun_out/launches_c5.csv python bench.py --config config5 --nt 12 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_list.log 2>&1
