mkdir -p gpurun_out
bash tools/gpu_round.sh
N=/usr/local/cuda/bin/ncu
timeout 600 $N --metrics gpu__time_duration.sum --clock-control none --csv -c 600 --log-file gpurun_out/launches_c2_final.csv python bench.py --config config2 --nt 200 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_c2_list.log 2>&1
timeout 1200 $N --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_scm3d<\(int\)3, \(int\)0>' -c 1 -o gpurun_out/scm3d_step_final python tools/step_bench.py config5 3 1 > gpurun_out/ncu_c5_final.log 2>&1
