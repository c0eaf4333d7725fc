mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_imex.py tests/test_gpu_elastic.py -x -q > gpurun_out/t4.log 2>&1; echo "exit $?" >> gpurun_out/t4.log
for q in 0.97 0.9 0.75; do
WAVECELL_B200_TRSV_Q=$q timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:trsv' -c 8 --log-file gpurun_out/launches_trsv_$q.csv python tools/imex_bench.py 1024 3 > gpurun_out/ncu_trsv_$q.log 2>&1
done
timeout 600 python tools/imex_bench.py 1024 200 > gpurun_out/imex_new.log 2>&1
