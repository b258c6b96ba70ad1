#!/bin/bash
# occupancy experiment for the cooperative kernel (64 registers, 2 CTAs/SM) + per-sweep trace
mkdir -p gpurun_out/r2j
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
bash tools/build_variant.sh /tmp/libhj_minb2.so -DHJ_COOP_MINB32=2 > gpurun_out/r2j/build_variant.log 2>&1; echo "variant rc=$?"
for lib in "" /tmp/libhj_minb2.so; do
  echo "== lib ${lib:-default}"
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_solve.py 3 f32 field_coop fine 2
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 3 2 | cut -c1-120
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 2 3 | cut -c1-120
  HJ_LIB_PATH=$lib timeout 300 python tools/prof_isa.py 4 2 | cut -c1-120
done > gpurun_out/r2j/occupancy.txt 2>&1
cat gpurun_out/r2j/occupancy.txt
timeout 300 python tools/coop_trace.py 3 > gpurun_out/r2j/coop_trace_c3.txt 2>&1; echo "trace rc=$?"; tail -30 gpurun_out/r2j/coop_trace_c3.txt
