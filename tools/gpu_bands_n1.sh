# The row-band / NCCL path at N=1 under torchrun (exchange + interior/edge
# launches), beside the whole-frame line, for 4K 4 spp and 8K.
for w in 4k4spp 8k; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --bands --workload $w --steps 16 --warmup 4 > gpurun_out/bench_bands_$w.log 2>&1; echo bands_$w=$?
done
