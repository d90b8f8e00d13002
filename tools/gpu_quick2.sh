#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "every_colour" > gpurun_out/pytest_colour.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_colour.log
