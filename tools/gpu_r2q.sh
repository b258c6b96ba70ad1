#!/bin/bash
mkdir -p gpurun_out/r2q
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "coop or segmented or sweep_kernels or partitioned or end_to_end or stops_inside" > gpurun_out/r2q/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r2q/pytest.log
for r in 1 2; do
timeout 300 python tools/prof_solve.py 3 f32 field_coop fine 2 | cut -c1-100
timeout 300 python tools/prof_isa.py 3 2 | grep wall | cut -c1-100
timeout 300 python tools/prof_isa.py 2 3 | grep wall | cut -c1-100
timeout 300 python tools/prof_isa.py 4 2 | grep wall | cut -c1-100
done
