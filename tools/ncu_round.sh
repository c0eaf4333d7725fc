#!/bin/bash
# ncu pass: launch lists (cold, serialised) and full captures of the top kernels.
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
L="--metrics gpu__time_duration.sum --clock-control none --csv"
if [[ "${WHAT:-5}" == *5* ]]; then
timeout 900 $NCU $L -c 2000 --log-file gpurun_out/launches_c5.csv python bench.py --config config5 --nt 4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_list.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_scm3d<3, 0>' -c 1 -o gpurun_out/scm3d_step python bench.py --config config5 --nt 4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_full.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_cut_pre' -s 3 -c 1 -o gpurun_out/cut_pre python bench.py --config config5 --nt 4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_cut.log 2>&1
fi
if [[ "${WHAT:-4}" == *4* ]]; then
timeout 900 $NCU $L -c 3000 --log-file gpurun_out/launches_c4.csv python tools/imex_bench.py 1024 10 > gpurun_out/ncu_c4_list.log 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_trsv_comp' -s 4 -c 2 -o gpurun_out/trsv python tools/imex_bench.py 1024 4 > gpurun_out/ncu_c4_full.log 2>&1
fi
