#!/bin/bash
# ncu evidence pass (one GPU): per configuration a launch list of the stepping
# loop (gpu__time_duration.sum, cold and serialised: shares, not absolutes) and
# one --set full capture of the dominant kernel.  Outputs in gpurun_out/.
mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
L="--metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled"
F="--set full --clock-control none --import-source on --kernel-name-base demangled -f"
B="--steps 1 --warmup 0 --no-cpu --no-e2e --no-secondary"
# config 2 (default bench workload, 64 of its 2000 time steps)
timeout 600 $N $L -k 'regex:k_scm2d|k_cdm|k_gather|k_scatter' -c 200 --log-file gpurun_out/launches_c2.csv python bench.py --config config2 --nt 64 $B > gpurun_out/ncu_c2_list.log 2>&1
timeout 600 $N $F -k 'regex:k_scm2d<.*4,.*0>' -s 30 -c 1 -o gpurun_out/scm2d_step python bench.py --config config2 --nt 64 $B > gpurun_out/ncu_c2_full.log 2>&1
# config 3
timeout 600 $N $L -k 'regex:k_sell<.*1>|k_cdm|k_gather|k_scatter' -c 200 --log-file gpurun_out/launches_c3.csv python bench.py --config config3 --nt 64 $B > gpurun_out/ncu_c3_list.log 2>&1
timeout 600 $N $F -k 'regex:k_sell<.*1>' -s 30 -c 1 -o gpurun_out/sell_step python bench.py --config config3 --nt 64 $B > gpurun_out/ncu_c3_full.log 2>&1
# config 4 (IMEX loop kernels)
timeout 900 $N $L -k 'regex:trsv|k_c_|_rows|k_rc_|ela2d<.*5,.*0>|k_imex|k_state' -s 60 -c 300 --log-file gpurun_out/launches_c4.csv python tools/imex_bench.py 1024 40 > gpurun_out/ncu_c4_list.log 2>&1
timeout 900 $N $F -k 'regex:k_trsv_ring' -s 6 -c 1 -o gpurun_out/trsv_ring python tools/imex_bench.py 1024 6 > gpurun_out/ncu_c4_trsv.log 2>&1
timeout 900 $N $F -k 'regex:ela2d<.*5,.*0>' -s 4 -c 1 -o gpurun_out/ela2d_step python tools/imex_bench.py 1024 6 > gpurun_out/ncu_c4_ela.log 2>&1
# config 5 (the list holds the power iteration too; tools/launch_summary.py --step keeps the stepping loop)
timeout 900 $N $L -k 'regex:k_scm3d|k_cut_pre' -c 6000 --log-file gpurun_out/launches_c5.csv python bench.py --config config5 --nt 12 $B > gpurun_out/ncu_c5_list.log 2>&1
timeout 900 $N $F -k 'regex:k_scm3d<.*3,.*0>' -s 2 -c 1 -o gpurun_out/scm3d_step python bench.py --config config5 --nt 6 $B > gpurun_out/ncu_c5_full.log 2>&1
