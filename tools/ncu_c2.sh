#!/bin/bash
# ncu pass for config 2: full capture of the 2D step kernel (a launch well inside the run)
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_scm2d<.*4,.*0>' -s 30 -c 1 -f -o gpurun_out/scm2d_step python bench.py --config config2 --nt 64 --steps 1 --warmup 0 --no-cpu --no-e2e --no-secondary > gpurun_out/ncu_c2_full.log 2>&1
