# Interleaved A/B of the kernel variants in build/var: R rounds, each variant
# once per round in a fresh process; then the GPU suite and the golden margin
# check on every variant.  usage: bash tools/ab_rounds.sh [R]
R=${1:-3}
rm -f gpurun_out/ab.log
for r in $(seq $R); do
  for so in build/var/libpgg_*.so; do
    v=$(basename $so .so)
    PGG_LIB=$PWD/$so timeout 300 python bench.py --steps 96 --warmup 16 --no-cpu-baseline --no-e2e --no-frame-loop \
      2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],5), d['clocks']['sm_mhz'])" >> gpurun_out/ab.log
  done
done
for so in build/var/libpgg_*.so; do
  v=$(basename $so .so)
  PGG_LIB=$PWD/$so timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pt_$v.log 2>&1; echo "tests $v rc=$?" >> gpurun_out/ab.log
  PGG_LIB=$PWD/$so timeout 300 python tools/margin_check.py > gpurun_out/margin_$v.log 2>&1; echo "margin $v rc=$?" >> gpurun_out/ab.log
done
