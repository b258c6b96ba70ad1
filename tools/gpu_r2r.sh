#!/bin/bash
mkdir -p gpurun_out/r2r
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 compute-sanitizer --tool memcheck --show-backtrace device python -m pytest tests/test_gpu_parity.py -x -q -k "list_mode and dubins" > gpurun_out/r2r/sanitizer.log 2>&1; echo "rc=$?"
grep -m 30 -E "Invalid|at |by thread|Address" gpurun_out/r2r/sanitizer.log | head -40
