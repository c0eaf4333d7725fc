mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_iga.py tests/test_gpu_timeint.py tests/test_gpu_dist.py -x -q > gpurun_out/t15.log 2>&1; echo "exit $?" >> gpurun_out/t15.log
timeout 300 python tools/step_bench.py config2 1000 3 > gpurun_out/t15_steps.log 2>&1
WAVECELL_B200_PDL=0 timeout 300 python tools/step_bench.py config2 1000 3 >> gpurun_out/t15_steps.log 2>&1
timeout 900 python bench.py --config config3 --no-cpu --no-e2e > gpurun_out/b3pdl.json 2> gpurun_out/b3pdl.err
