mkdir -p gpurun_out
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k 'regex:k_sell<\(bool\)1>' -s 5 -c 1 -o gpurun_out/sell_step python bench.py --config config3 --nt 20 --steps 1 --warmup 0 --no-cpu --no-e2e > gpurun_out/ncu_sell.log 2>&1
