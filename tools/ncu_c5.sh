#!/bin/bash
# ncu pass for config 5: full capture of the 3D step kernel (third step launch)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_scm3d<.*3,.*0>' -s 2 -c 1 -f -o gpurun_out/scm3d_step python bench.py --config config5 --nt 6 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_full.log 2>&1
