mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_dist.py tests/test_gpu_timeint.py -x -q > gpurun_out/t3v.log 2>&1; echo "exit $?" >> gpurun_out/t3v.log
for v in libwavecell_b200.so libwavecell_b200_noreuse.so libwavecell_b200_wy7.so libwavecell_b200_wy7nr.so; do
  WAVECELL_B200_LIB=$v timeout 300 python tools/step_bench.py config5 20 2 >> gpurun_out/t3v_steps.log 2>&1; echo "$v" >> gpurun_out/t3v_steps.log
done
timeout 300 python tools/step_bench.py config2 500 3 >> gpurun_out/t3v_steps.log 2>&1
WAVECELL_B200_NO_MINV_TAB=1 timeout 300 python tools/step_bench.py config2 500 3 >> gpurun_out/t3v_steps.log 2>&1
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv -k 'regex:trsv|ela2d|k_c_|perm|gather_rows' -c 400 --log-file gpurun_out/launches_c4b.csv python tools/imex_bench.py 1024 5 > gpurun_out/ncu_c4b.log 2>&1
