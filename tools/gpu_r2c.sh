#!/bin/bash
mkdir -p gpurun_out/r2c
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2c/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/r2c/pytest_gpu.log
