# A/B the variants in build/var: bench (fresh process each, twice, interleaved) + golden margins
set -u
: > gpurun_out/ab.log
for rep in 1 2; do
for so in build/var/libpgg_*.so; do
  echo "== $so" >> gpurun_out/ab.log
  PGG_LIB=$PWD/$so timeout 300 python bench.py --steps 96 --warmup 16 --no-cpu-baseline --no-e2e --no-frame-loop 2>&1 | \
    python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ms', round(d['ms_per_step'],4), 'kernel', round(d['roofline']['kernel_ms'],4))" >> gpurun_out/ab.log 2>&1
done
done
for so in build/var/libpgg_*.so; do
  echo "== margins $so" >> gpurun_out/ab.log
  PGG_LIB=$PWD/$so timeout 300 python tools/margin_check.py >> gpurun_out/ab.log 2>&1
done
