#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
#timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep_kernels or edge_cases or stops_inside or partitioned" > gpurun_out/pytest9.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest9.log
( timeout 300 python tools/prof_solve.py 2 f32 local_tb fine 2
  timeout 300 python tools/prof_solve.py 2 f32 local_tb coarse 2
  timeout 300 python tools/prof_solve.py 2 f64 local_tb fine 1 ) > gpurun_out/solve11.txt 2>&1
cat gpurun_out/solve11.txt
python tools/prof_solve.py 2 f32 local_tb fine 1 > gpurun_out/plain11.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_tb -s 40 -c 2 -o gpurun_out/prof_tb6 python tools/prof_solve.py 2 f32 local_tb fine 1 > gpurun_out/ncu11.log 2>&1
echo "ncu rc=$?"
