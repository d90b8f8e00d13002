#!/bin/bash
# multi-GPU gpurun: N-rank bench (weak scaling, C2 per rank) + C3 strong scaling
mkdir -p gpurun_out
N=${N:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus $N --steps 30 --warmup 3 > gpurun_out/bench_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n$N.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29513 \
  bench.py --gpus $N --steps 30 --warmup 3 --no-gather --no-e2e > gpurun_out/bench_n${N}_nogather.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n${N}_nogather.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --gpus $N --config C3 --steps 2 --warmup 1 > gpurun_out/bench_c3_n$N.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3_n$N.log
if [ "$N" = "2" ]; then
  timeout 900 python bench.py --config C3 --steps 2 --warmup 1 > gpurun_out/bench_c3_n1.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3_n1.log
fi
