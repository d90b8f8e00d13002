#!/bin/bash
# packed streaming batches (C5) + unpack4x K1 variants
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_nv12.py -x -q -k "packed_batches or every_k1_config or mixed_sources or golden" > gpurun_out/pytest_batch.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_batch.log
timeout 1200 python bench.py --config C5 --steps 2 --warmup 1 > gpurun_out/bench_C5_n1_batch.log 2>&1
K1_CFGS=49,56,57 timeout 900 python tools/k1_ab.py 18000 5 > gpurun_out/k1_ab5.log 2>&1
echo done >> gpurun_out/k1_ab5.log
