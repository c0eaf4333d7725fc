mkdir -p gpurun_out
N=/usr/local/cuda/bin/ncu
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 900 python bench.py --config config2 > gpurun_out/bench_config2.json 2> gpurun_out/bench_config2.err
timeout 900 python bench.py --config config4 > gpurun_out/bench_config4.json 2> gpurun_out/bench_config4.err
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv -c 600 --log-file gpurun_out/launches_c2.csv python bench.py --config config2 --nt 200 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c2_list.log 2>&1
timeout 600 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_scm2d<\(int\)4, \(int\)0>' -s 20 -c 1 -o gpurun_out/scm2d_step_v2 python bench.py --config config2 --nt 40 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c2_full.log 2>&1
