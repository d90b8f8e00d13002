# ncu evidence for profiles/r02 (one ncu use per gpurun call: this script is one call).
# 1) launch list of the default bench command, 2) --set full of K1, K1-NV12, K4, K3.
mkdir -p gpurun_out/r2/ncu
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
NCU=/usr/local/cuda/bin/ncu
python tools/k1_one.py 2000 > gpurun_out/r2/ncu/plain_one.log 2>&1 && \
$NCU --set full --clock-control none --import-source on \
     -k regex:"k1_hist_kernel|k1_nv12_kernel|k4_sample_kernel|k3_rounds_kernel" -s 0 -c 12 \
     -o gpurun_out/r2/ncu/full python tools/k1_one.py 2000 > gpurun_out/r2/ncu/full.log 2>&1
echo "full rc=$?"
python bench.py --steps 3 --warmup 3 --no-c3 --no-cpu > gpurun_out/r2/ncu/plain_bench.log 2>&1 && \
$NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
     --log-file gpurun_out/r2/ncu/launches.csv python bench.py --steps 3 --warmup 3 --no-c3 --no-cpu \
     > gpurun_out/r2/ncu/launches.log 2>&1
echo "launches rc=$?"
