mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
timeout 400 python tools/imex_bench.py 256 3 > gpurun_out/plain4.log 2>&1 || exit 1
K='regex:trsv|ela2d<\(int\)5, \(int\)0>|k_c_|gather_rows|perm_rows|ela2d<\(int\)5, \(int\)1>'
timeout 900 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "$K" -s 200 -c 60 --log-file gpurun_out/launches_c4_final.csv python tools/imex_bench.py 1024 4 > gpurun_out/ncu_c4_list.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_trsv_comp' -s 4 -c 1 -o gpurun_out/trsv_final python tools/imex_bench.py 1024 2 > gpurun_out/ncu_trsv_final.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ela2d<\(int\)5, \(int\)0>' -s 2 -c 1 -o gpurun_out/ela2d_step python tools/imex_bench.py 1024 2 > gpurun_out/ncu_ela2d.log 2>&1
