#!/bin/bash
# 4-GPU box: NV12 weak scaling (C2 NV12 per GPU) and frame-sharded NV12 at N = 2, 4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for N in 4 2; do
  DEVS=$(seq -s, 0 $((N-1)))
  CUDA_VISIBLE_DEVICES=$DEVS timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 2962$N bench.py --gpus $N --format nv12 --no-cpu --steps 30 --warmup 3 \
    > gpurun_out/bench_nv12_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_nv12_n$N.log
  CUDA_VISIBLE_DEVICES=$DEVS timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 2963$N bench.py --gpus $N --format nv12 --shard-frames --steps 30 --warmup 3 \
    > gpurun_out/bench_shard_nv12_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shard_nv12_n$N.log
done
python bench.py --format nv12 --no-cpu > gpurun_out/bench_nv12_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_nv12_n1.log
python bench.py --format nv12 --shard-frames > gpurun_out/bench_shard_nv12_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_shard_nv12_n1.log
