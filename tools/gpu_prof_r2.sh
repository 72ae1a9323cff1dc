# ncu --set full capture of the headline kernel (one launch, steady state)
# plus the launch list of the bench command; run only after bench exits 0.
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/bench_small.log 2>&1; echo bench=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_guiding_pass -s 10 -c 1 -o gpurun_out/prof_${1:-r2} -f \
  python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
