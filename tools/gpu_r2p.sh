#!/bin/bash
mkdir -p gpurun_out/r2p
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh /tmp/libhj_u8.so -DHJ_COL2_ROW_UNROLL=8 > /dev/null 2>&1; echo "v8 rc=$?"
bash tools/build_variant.sh /tmp/libhj_u2.so -DHJ_COL2_ROW_UNROLL=2 > /dev/null 2>&1; echo "v2 rc=$?"
for r in 1 2; do
for lib in "" /tmp/libhj_u8.so /tmp/libhj_u2.so; do echo "lib ${lib:-default}"; HJ_LIB_PATH=$lib timeout 600 python tools/prof_solve.py 5 f32 field_col fine 1 200 | cut -c1-100; done
HJ_NO_COL2=1 timeout 600 python tools/prof_solve.py 5 f32 field_col fine 1 200 | cut -c1-100
done
