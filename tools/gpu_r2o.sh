#!/bin/bash
mkdir -p gpurun_out/r2o
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "field_col or sweep_kernels or partitioned or end_to_end" > gpurun_out/r2o/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2o/pytest.log
for e in "" 1; do HJ_NO_COL2=$e timeout 600 python tools/prof_solve.py 5 f32 field_col fine 2 200 | cut -c1-150; done
timeout 900 python tools/prof_isa.py 5 | cut -c1-150
python tools/prof_solve.py 5 f32 field_col fine 1 20 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d_col2 --launch-skip 10 --launch-count 1 \
    -o gpurun_out/r2o/ncu_c5_col2 python tools/prof_solve.py 5 f32 field_col fine 1 20 > gpurun_out/r2o/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_roofline.py gpurun_out/r2o/ncu_c5_col2.ncu-rep c5_regulator_16385 gpurun_out/r2o/ncu_roofline_c5_regulator_16385.json k_sweep_field2d_col2 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|dram_gbs|long_sc|wait"
