#!/bin/bash
# call 2: ALU microbenchmark, new kernel tests, solve timings, ncu --set full of the sweeps
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_alu.cu && /tmp/ub > gpurun_out/ubench_alu.txt 2>&1
cat gpurun_out/ubench_alu.txt
python -c "import __graft_entry__ as g; g.build()"
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep_kernels or refuses or solve_matches" > gpurun_out/pytest2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest2.log
for k in local_scalar local_packed generic; do timeout 300 python tools/prof_solve.py 2 f32 $k fine 2; done > gpurun_out/solve_c2.txt 2>&1
timeout 300 python tools/prof_solve.py 2 f32 auto coarse 2 >> gpurun_out/solve_c2.txt 2>&1
timeout 300 python tools/prof_solve.py 4 f32 auto fine 1 40 > gpurun_out/solve_c4.txt 2>&1
cat gpurun_out/solve_c2.txt gpurun_out/solve_c4.txt
python tools/prof_solve.py 2 f32 local_scalar fine 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d -s 400 -c 2 -o gpurun_out/prof_local_scalar python tools/prof_solve.py 2 f32 local_scalar fine 1 > gpurun_out/ncu1.log 2>&1
python tools/prof_solve.py 2 f32 local_packed fine 1 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_x2 -s 400 -c 2 -o gpurun_out/prof_local_packed python tools/prof_solve.py 2 f32 local_packed fine 1 > gpurun_out/ncu2.log 2>&1
python tools/prof_solve.py 4 f32 auto fine 1 12 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_sweep_generic -s 10 -c 1 -o gpurun_out/prof_generic_c4 python tools/prof_solve.py 4 f32 auto fine 1 12 > gpurun_out/ncu3.log 2>&1
echo "ncu done rc=$?"; ls gpurun_out
