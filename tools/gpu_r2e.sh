#!/bin/bash
mkdir -p gpurun_out/r2e
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2e/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2e/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -45 gpurun_out/r2e/pytest_gpu.log
timeout 600 python tools/prof_isa.py 5 > gpurun_out/r2e/isa_c5.txt 2>&1; echo "isa c5 rc=$?"; tail -5 gpurun_out/r2e/isa_c5.txt
