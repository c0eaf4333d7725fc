mkdir -p gpurun_out
timeout 300 python tools/e2e_profile.py config2 2000 > gpurun_out/e2e.log 2>&1
timeout 900 python bench.py --config config4 --steps 3 --warmup 1 --no-cpu > gpurun_out/b4n1.json 2> gpurun_out/b4n1.err
