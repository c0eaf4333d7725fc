mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
timeout 600 python tools/imex_bench.py 256 3 > gpurun_out/plain.log 2>&1 || exit 1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_ela2s' -c 1 -o gpurun_out/ela2s python tools/imex_bench.py 1024 2 > gpurun_out/ncu_ela2s.log 2>&1
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_trsv_comp' -s 2 -c 1 -o gpurun_out/trsv2 python tools/imex_bench.py 1024 2 > gpurun_out/ncu_trsv2.log 2>&1
