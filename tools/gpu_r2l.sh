#!/bin/bash
# A/B on one box: vectorised seg table vs scalar
mkdir -p gpurun_out/r2l
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh /tmp/libhj_segvec0.so -DHJ_SEG_VEC=0 > /dev/null 2>&1; echo "variant rc=$?"
for r in 1 2; do for lib in "" /tmp/libhj_segvec0.so; do
  echo "== lib ${lib:-default} rep $r"
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_solve.py 3 f32 field_coop fine 2 | cut -c1-100
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 3 2 | grep wall | cut -c1-100
done; done
