#!/bin/bash
mkdir -p gpurun_out/r2s
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh /tmp/libhj_dbg.so -DHJ_DEBUG_BOUNDS > gpurun_out/r2s/build.log 2>&1; echo "dbg rc=$?"
HJ_LIB_PATH=/tmp/libhj_dbg.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "list_mode and dubins" > gpurun_out/r2s/dbg.log 2>&1; echo "dbg test rc=$?"
grep -m5 "HJ_DEBUG\|Error\|passed\|failed" gpurun_out/r2s/dbg.log
for m in 0 1; do HJ_COOP_LIST=$m timeout 300 python tools/prof_solve.py 4 f32 dubins_coop fine 1 2>&1 | tail -2 | cut -c1-150; done
