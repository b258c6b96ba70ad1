#!/bin/bash
mkdir -p gpurun_out/r2g
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "segmented or sweep_kernels or coop_list or partitioned" > gpurun_out/r2g/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2g/pytest.log
for e in 1 ""; do HJ_NO_SEG=$e timeout 600 python bench.py --steps 2 --no-cpu-baseline > gpurun_out/r2g/bench_c3_seg$e.json 2>&1; echo "bench rc=$?"; python -c "
import json,sys; d=json.loads(open('gpurun_out/r2g/bench_c3_seg$e.json').read().splitlines()[-1]); print('NO_SEG=$e', d['ms_per_step'], d['stages_ms'], d['roofline']['frac'])"; done
python tools/prof_step.py 3 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 3 --launch-count 1 \
    -o gpurun_out/r2g/ncu_c3_fine python tools/prof_step.py 3 > gpurun_out/r2g/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_roofline.py gpurun_out/r2g/ncu_c3_fine.ncu-rep c3_zermelo_4097 gpurun_out/r2g/ncu_roofline_c3_zermelo_4097.json k_sweep_local2d_coop 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|barrier|wait"
