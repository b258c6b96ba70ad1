#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
python tools/prof_solve.py 2 f32 local_tb fine 1 > gpurun_out/plain5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_tb -s 40 -c 2 -o gpurun_out/prof_tb python tools/prof_solve.py 2 f32 local_tb fine 1 > gpurun_out/ncu6.log 2>&1
echo "ncu rc=$?"
