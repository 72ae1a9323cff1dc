python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 1200 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_guiding_pass -s 10 -c 1 -o gpurun_out/prof_r1n python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu2=$?
