# one ncu --set full capture of k_guiding_pass per variant library in build/var
set -u
for so in build/var/libpgg_*.so; do
  n=$(basename $so .so)
  PGG_LIB=$PWD/$so timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_guiding_pass -s 10 -c 1 -o gpurun_out/ab_$n -f \
    python bench.py --steps 16 --warmup 8 --no-cpu-baseline --no-e2e --no-frame-loop > gpurun_out/ncu_ab_$n.log 2>&1; echo $n=$?
done
