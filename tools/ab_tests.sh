# A/B timing plus the full GPU parity suite against every variant in build/var
for so in build/var/libpgg_*.so; do
  echo "== $so" >> gpurun_out/ab.log
  PGG_LIB=$PWD/$so timeout 300 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e --no-frame-loop >> gpurun_out/ab.log 2>&1
  PGG_LIB=$PWD/$so timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pt_$(basename $so .so).log 2>&1; echo "tests $(basename $so) rc=$?" >> gpurun_out/ab.log
done
