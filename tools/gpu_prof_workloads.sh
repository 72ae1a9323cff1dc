# one ncu --set full capture of k_guiding_pass per bench workload (for profiles/traffic.json)
for w in 4k4spp 8k; do
  timeout 600 python bench.py --workload $w --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/bench_prof_$w.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none -k regex:k_guiding_pass -s 6 -c 1 -o gpurun_out/prof_$w \
    python bench.py --workload $w --steps 8 --warmup 4 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/ncu_$w.log 2>&1; echo $w=$?
done
