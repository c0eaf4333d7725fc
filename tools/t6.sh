mkdir -p gpurun_out
K='regex:trsv'
for q in 1.0 0.99; do
WAVECELL_B200_TRSV_Q=$q timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --kernel-name-base demangled -k "$K" -c 12 --log-file gpurun_out/launches_trsv_q$q.csv python tools/imex_bench.py 1024 3 > gpurun_out/ncu_trsv_q$q.log 2>&1
done
for c in config2 config3 config4 config5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "$c exit $?" >> gpurun_out/bench_status.txt
done
