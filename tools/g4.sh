mkdir -p gpurun_out
timeout 900 python bench.py --config config4 > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
N=/usr/local/cuda/bin/ncu
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:trsv|k_c_|_rows|k_rc_|ela2d<.*5,.*0>|k_imex|k_state' -s 60 -c 300 --log-file gpurun_out/launches_c4.csv python tools/imex_bench.py 1024 40 > gpurun_out/ncu_c4_list.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -f -k 'regex:ela2d<.*5,.*0>' -s 4 -c 1 -o gpurun_out/ela2d_step python tools/imex_bench.py 1024 6 > gpurun_out/ncu_c4_ela.log 2>&1
