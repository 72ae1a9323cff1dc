# A/B the kernel variants in build/var (same bench, fresh process each)
for so in build/var/libpgg_*.so; do
  echo "== $so" >> gpurun_out/ab.log
  PGG_LIB=$PWD/$so timeout 300 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e >> gpurun_out/ab.log 2>&1
done
