mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py tests/test_gpu_timeint.py tests/test_gpu_scm.py -x -q > gpurun_out/t4.log 2>&1; echo "exit $?" >> gpurun_out/t4.log
K='regex:trsv|ela2s|ela2d<\(int\)5, \(int\)0>'
for t in ${THREADS:-64 128 256}; do
WAVECELL_B200_TRSV_THREADS=$t timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "$K" -c 12 --log-file gpurun_out/launches_trsv_t$t.csv python tools/imex_bench.py 1024 3 > gpurun_out/ncu_trsv_t$t.log 2>&1
done
WAVECELL_B200_TILE_ELASTIC=1 timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "$K" -c 12 --log-file gpurun_out/launches_ela_tile.csv python tools/imex_bench.py 1024 3 > gpurun_out/ncu_ela_tile.log 2>&1
timeout 600 python tools/imex_bench.py 1024 200 > gpurun_out/imex_new.log 2>&1
timeout 300 python tools/step_bench.py config5 20 2 > gpurun_out/s5.log 2>&1
