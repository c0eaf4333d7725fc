mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
WAVECELL_B200_NO_IMEX_OVERLAP=1 timeout 900 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:ela2d<.*5,.*0>' -s 3 -c 1 -f -o gpurun_out/ela2d_step python tools/imex_bench.py 1024 6 > gpurun_out/ncu_ela2d.log 2>&1
