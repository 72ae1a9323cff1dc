# The bench lines only (both arms, 1080p headline + 4K / 8K), for profiles/
set -u
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1; echo bench_ref=$?
timeout 600 python bench.py --workload 4k4spp --steps 32 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_4k.log 2>&1; echo b4k=$?
timeout 600 python bench.py --workload 8k --steps 16 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/bench_8k.log 2>&1; echo b8k=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-frame-loop > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
