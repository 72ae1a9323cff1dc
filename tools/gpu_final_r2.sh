# Round-2 evidence: build + smoke, GPU tests (reports under gpurun_out/),
# the bench lines (driver form, reference arm, 4K 4 spp, 8K 64-frame
# sequence), the ncu launch list of the bench command and --set full
# captures of the pass at 1080p / 4K 4 spp / 8K (traffic + instructions).
set -u
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
rm -f gpurun_out/hazards.json
PGG_REPORT_DIR=gpurun_out timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 600 python bench.py --workload 4k4spp --steps 32 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_4k.log 2>&1; echo b4k=$?
timeout 900 python bench.py --workload 8k --seq 64 > gpurun_out/bench_8k_seq64.log 2>&1; echo seq64=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"^k_" -c 400 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 4 --warmup 3 --no-cpu-baseline --no-frame-loop > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_guiding_pass -s 10 -c 1 -f \
  -o gpurun_out/prof_final python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/ncu_full.log 2>&1; echo ncu_full=$?
timeout 900 ncu --set full --clock-control none -k regex:k_guiding_pass -s 10 -c 1 -f \
  -o gpurun_out/prof_4k4spp python bench.py --workload 4k4spp --steps 12 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/ncu_4k.log 2>&1; echo ncu_4k=$?
timeout 900 ncu --set full --clock-control none -k regex:k_guiding_pass -s 10 -c 1 -f \
  -o gpurun_out/prof_8k python bench.py --workload 8k --steps 12 --warmup 4 --no-cpu-baseline --no-e2e > gpurun_out/ncu_8k.log 2>&1; echo ncu_8k=$?
