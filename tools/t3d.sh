mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_scm.py tests/test_gpu_dist.py tests/test_gpu_imex.py tests/test_gpu_elastic.py -x -q > gpurun_out/t3d.log 2>&1; echo "exit $?" >> gpurun_out/t3d.log
timeout 600 python bench.py --config config5 --steps 3 --warmup 1 --no-cpu > gpurun_out/b5new.json 2> gpurun_out/b5new.err
timeout 600 python tools/imex_bench.py 1024 200 > gpurun_out/imex_new.log 2>&1
if [ -n "$NCU" ]; then
timeout 1200 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k 'regex:k_scm3d<\(int\)3, \(int\)0>' --kernel-name-base demangled -c 1 -o gpurun_out/scm3d_step python bench.py --config config5 --nt 4 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c5_full.log 2>&1
fi
