python -c "import __graft_entry__ as g; g.build()"
PGG_SPLIT=1 timeout 600 python bench.py --steps 8 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_split.log 2>&1 && \
PGG_SPLIT=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_stage1" -s 8 -c 1 -o gpurun_out/prof_stage1 python bench.py --steps 8 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/ncu_split.log 2>&1; echo rc=$?
