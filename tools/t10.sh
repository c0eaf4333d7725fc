mkdir -p gpurun_out
for v in libwavecell_b200.so libwavecell_b200_rpe4.so libwavecell_b200_rpe2.so libwavecell_b200_rpe3m3.so; do
  WAVECELL_B200_LIB=$v timeout 300 python tools/step_bench.py config2 1000 3 >> gpurun_out/t10.log 2>&1; echo "$v" >> gpurun_out/t10.log
done
