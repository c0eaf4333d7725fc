# bench lines of configs 3-5 (one GPU) into gpurun_out/
mkdir -p gpurun_out
for c in config3 config4 config5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err
  echo "$c exit $?" >> gpurun_out/bench_all.log
done
