#!/bin/bash
# A/B: warps per cooperative CTA (fp32): 16 (default), 20, 24
mkdir -p gpurun_out/r2u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh /tmp/libhj_nw20.so -DHJ_COOP_NW32=20 > /dev/null 2>&1; echo "nw20 rc=$?"
bash tools/build_variant.sh /tmp/libhj_nw24.so -DHJ_COOP_NW32=24 > /dev/null 2>&1; echo "nw24 rc=$?"
for r in 1 2; do for lib in "" /tmp/libhj_nw20.so /tmp/libhj_nw24.so; do
  echo "== ${lib:-default} rep $r"
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_solve.py 3 f32 field_coop fine 1 | cut -c1-100
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 3 2 | grep wall | tail -1 | cut -c1-100
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 2 3 | grep wall | tail -1 | cut -c1-100
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 4 2 | grep wall | tail -1 | cut -c1-100
done; done
