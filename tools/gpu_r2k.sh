#!/bin/bash
mkdir -p gpurun_out/r2k
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "segmented or sweep_kernels or coop or partitioned or end_to_end" > gpurun_out/r2k/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r2k/pytest.log
for c in 3 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/r2k/bench_c$c.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/r2k/bench_c$c.json').read().splitlines()[-1]); print('c$c', round(d['ms_per_step'],2), d['step_ms'], d['stages_ms'])"; done
timeout 300 python tools/prof_solve.py 3 f32 field_coop fine 2
