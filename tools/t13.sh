mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_timeint.py tests/test_gpu_scm.py tests/test_gpu_imex.py tests/test_gpu_iga.py -x -q > gpurun_out/t13.log 2>&1; echo "exit $?" >> gpurun_out/t13.log
timeout 300 python tools/e2e_profile.py config2 2000 > gpurun_out/e2e.log 2>&1
timeout 900 python bench.py --config config2 --no-cpu > gpurun_out/b2.json 2> gpurun_out/b2.err
