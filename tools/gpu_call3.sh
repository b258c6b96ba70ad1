#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep_kernels or refuses or edge_cases or solve_matches" > gpurun_out/pytest3.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest3.log
( timeout 300 python tools/prof_solve.py 2 f32 field2d fine 1
  timeout 300 python tools/prof_solve.py 3 f32 auto fine 1
  timeout 300 python tools/prof_solve.py 4 f32 auto fine 2
  timeout 300 python tools/prof_solve.py 4 f32 generic fine 1 40
  timeout 300 python tools/prof_solve.py 5 f32 auto fine 1 100
  timeout 300 python tools/prof_solve.py 5 f32 auto coarse 1 ) > gpurun_out/solve3.txt 2>&1
cat gpurun_out/solve3.txt
python tools/prof_solve.py 5 f32 auto fine 1 6 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d -s 3 -c 1 -o gpurun_out/prof_field2d_c5 python tools/prof_solve.py 5 f32 auto fine 1 6 > gpurun_out/ncu4.log 2>&1
python tools/prof_solve.py 4 f32 auto fine 1 12 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_dubins -s 10 -c 1 -o gpurun_out/prof_dubins_c4 python tools/prof_solve.py 4 f32 auto fine 1 12 > gpurun_out/ncu5.log 2>&1
echo "ncu rc=$?"
