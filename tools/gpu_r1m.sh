python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_bands.py -q > gpurun_out/pytest_bands.log 2>&1; echo bands=$?
timeout 900 python bench.py --workload 4k4spp --steps 32 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_4k.log 2>&1; echo b4k=$?
timeout 900 python bench.py --workload 8k --steps 16 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_8k.log 2>&1; echo b8k=$?
timeout 900 python bench.py --steps 160 --warmup 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_1080.log 2>&1; echo b1080=$?
