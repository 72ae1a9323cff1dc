# Round-2 bench lines: default (driver form), reference arm, 8K 64-frame sequence, 4K 4 spp, --gpus 2 error path
set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_default.log 2>&1; echo bench=$?
timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_ref.log 2>&1; echo ref=$?
timeout 900 python bench.py --workload 8k --seq 64 > gpurun_out/bench_8k_seq64.log 2>&1; echo seq64=$?
timeout 600 python bench.py --workload 4k4spp --steps 32 --warmup 8 --no-cpu-baseline --no-e2e > gpurun_out/bench_4k.log 2>&1; echo b4k=$?
timeout 120 python bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/bench_gpus2.log 2>&1; echo gpus2=$?
