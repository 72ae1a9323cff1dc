# A/B the render variants in build/var
for so in build/var/libpgg_*.so; do
  echo "== $so" >> gpurun_out/ab_render.log
  PGG_LIB=$PWD/$so timeout 300 python tools/bench_render.py --frames 16 --warmup 4 --cpu-sample 0 >> gpurun_out/ab_render.log 2>&1
done
