mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
for only in 0 1 8 148; do
WAVECELL_B200_TRSV_ONLY=$only timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k 'regex:trsv' -s 20 -c 6 --log-file gpurun_out/launches_only$only.csv python tools/imex_bench.py 1024 20 > gpurun_out/ncu_c4_list.log 2>&1
done
