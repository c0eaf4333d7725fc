mkdir -p gpurun_out
for v in libwavecell_b200.so libwavecell_b200_ela3.so libwavecell_b200_ela4.so; do
  WAVECELL_B200_LIB=$v timeout 400 python tools/imex_bench.py 1024 200 2>&1 | tail -1 >> gpurun_out/t17.log; echo "$v" >> gpurun_out/t17.log
done
