# N-GPU runs of bench.py (self-launching: one process per GPU over NCCL).
# usage: bash tools/gpu_multi.sh <N>     (logs in gpurun_out/r2/multi/)
N=$1
mkdir -p gpurun_out/r2/multi
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
nvidia-smi topo -m > gpurun_out/r2/multi/topo_n$N.txt 2>&1
export NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,COLL NCCL_DEBUG_FILE=gpurun_out/r2/multi/nccl_n$N.%h.%p.log
timeout 1200 python bench.py --gpus $N --steps 10 --warmup 3 --no-cpu > gpurun_out/r2/multi/bench_n$N.log 2> gpurun_out/r2/multi/bench_n$N.err
echo "bench n=$N rc=$?"; tail -c 600 gpurun_out/r2/multi/bench_n$N.log
timeout 900 python bench.py --gpus $N --shard-frames --steps 10 --warmup 3 > gpurun_out/r2/multi/shard_n$N.log 2> gpurun_out/r2/multi/shard_n$N.err
echo "shard n=$N rc=$?"; tail -c 400 gpurun_out/r2/multi/shard_n$N.log
timeout 1200 python bench.py --gpus $N --config C5 --steps 2 --warmup 1 > gpurun_out/r2/multi/c5_n$N.log 2> gpurun_out/r2/multi/c5_n$N.err
echo "c5 n=$N rc=$?"; tail -c 400 gpurun_out/r2/multi/c5_n$N.log
timeout 600 python bench.py --gpus $N --steps 10 --warmup 3 --no-cpu --no-gather --no-c3 --no-noise --no-e2e --sample-k 0 > gpurun_out/r2/multi/nogather_n$N.log 2> gpurun_out/r2/multi/nogather_n$N.err
echo "nogather n=$N rc=$?"; tail -c 300 gpurun_out/r2/multi/nogather_n$N.log
