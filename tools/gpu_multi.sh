#!/bin/bash
# multi-GPU gpurun: N-rank bench (weak scaling, C2 per rank) + C3/C4/C5 strong scaling
mkdir -p gpurun_out
N=${N:-2}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
nvidia-smi topo -m > gpurun_out/topo_$N.txt 2>&1
run() {  # name, port, args...
  local name=$1 port=$2; shift 2
  if [ "$N" = "1" ]; then
    timeout 1200 python bench.py "$@" > gpurun_out/$name.log 2>&1; echo "rc=$?" >> gpurun_out/$name.log
  else
    timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $port bench.py --gpus $N "$@" > gpurun_out/$name.log 2>&1; echo "rc=$?" >> gpurun_out/$name.log
  fi
}
if [ -z "$ONLY_CONFIGS" ]; then
run bench_n$N 29511 --steps 30 --warmup 3 ${BENCH_EXTRA}
run bench_shard_n$N 29514 --shard-frames --steps 30 --warmup 3
fi
for c in ${CONFIGS:-C3 C4 C5}; do
  run bench_${c}_n$N 29512 --config $c --steps 2 --warmup 1
done
