# A/B env variants of the same build
rm -f gpurun_out/ab.log
python -c "import __graft_entry__ as g; g.build()"
for v in "PGG_SPLIT=0" "PGG_SPLIT=1"; do
  echo "== $v" >> gpurun_out/ab.log
  env $v timeout 300 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e >> gpurun_out/ab.log 2>&1
done
PGG_SPLIT=1 timeout 600 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_split.log 2>&1; echo split_tests=$? >> gpurun_out/ab.log
