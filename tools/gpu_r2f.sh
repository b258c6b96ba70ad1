#!/bin/bash
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -q -k "multirank or partitioned or field_col or sweep_kernels or edge" > gpurun_out/r2f/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2f/pytest.log
for k in field2d field_col; do timeout 600 python tools/prof_solve.py 5 f32 $k fine 2 200; done > gpurun_out/r2f/solve_c5.txt 2>&1
cat gpurun_out/r2f/solve_c5.txt
timeout 600 python tools/prof_isa.py 5 > gpurun_out/r2f/isa_c5.txt 2>&1; echo "isa c5 rc=$?"; cat gpurun_out/r2f/isa_c5.txt
python tools/prof_solve.py 5 f32 field_col fine 1 20 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d_col --launch-skip 10 --launch-count 1 \
    -o gpurun_out/r2f/ncu_c5_col python tools/prof_solve.py 5 f32 field_col fine 1 20 > gpurun_out/r2f/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_roofline.py gpurun_out/r2f/ncu_c5_col.ncu-rep c5_regulator_16385 gpurun_out/r2f/ncu_c5_col.json k_sweep_field2d_col 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|dram_gbs"
