mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_imex_slabs.py tests/test_gpu_paper.py tests/test_gpu_tensor.py -m gpu -q --timeout 200 > gpurun_out/t4.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4.log
timeout 400 python tools/imex_bench.py 1024 200 > gpurun_out/imex_1024.log 2>&1
N=/usr/local/cuda/bin/ncu
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:trsv|k_c_|_rows|k_rc_|ela2d<.*5,.*0>|k_imex|k_state' -s 60 -c 300 --log-file gpurun_out/launches_c4.csv python tools/imex_bench.py 1024 40 > gpurun_out/ncu_c4_list.log 2>&1
timeout 600 python -m pytest tests/test_gpu_bench_parity.py -m gpu -q -k "config4" --timeout 300 > gpurun_out/t4b.log 2>&1; echo "pytest exit $?" >> gpurun_out/t4b.log
