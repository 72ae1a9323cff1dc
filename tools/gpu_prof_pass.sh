timeout 600 python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e > gpurun_out/bench_small.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_guiding_pass -s 10 -c 1 -o gpurun_out/prof_pass python bench.py --steps 64 --warmup 16 --no-cpu-baseline --no-e2e > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
