mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_trsv_ring' -s 6 -c 1 -f -o gpurun_out/trsv_ring python tools/imex_bench.py 1024 6 > gpurun_out/ncu_c4_trsv.log 2>&1
