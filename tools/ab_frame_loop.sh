# A/B of the whole-frame loop (bench_render stages + the bench frame_loop leg) over the libraries in build/var
rm -f gpurun_out/abr.log
for r in 1 2 3; do for so in build/var/libpgg_*.so; do v=$(basename $so .so)
  echo "== $v" >> gpurun_out/abr.log
  PGG_LIB=$PWD/$so timeout 300 python tools/bench_render.py --frames 16 --warmup 4 --cpu-sample 0 2>/dev/null | tail -1 >> gpurun_out/abr.log
  PGG_LIB=$PWD/$so timeout 300 python bench.py --steps 16 --warmup 4 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['frame_loop']['ms_per_frame'], d['frame_loop']['ms_per_frame_min_max'])" >> gpurun_out/abr.log
done; done
for so in build/var/libpgg_*.so; do v=$(basename $so .so)
  PGG_LIB=$PWD/$so timeout 900 python -m pytest tests/test_gpu_render.py tests/test_gpu_cli.py tests/test_gpu_acceptance.py tests/test_gpu_spec.py -q -x -p no:cacheprovider > gpurun_out/ptr_$v.log 2>&1; echo "render tests $v rc=$?" >> gpurun_out/abr.log
done
