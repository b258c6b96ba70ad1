#!/bin/bash
mkdir -p gpurun_out/r2h
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python tools/prof_isa.py 3 2 > gpurun_out/r2h/isa_c3_seg.txt 2>&1
HJ_NO_SEG=1 timeout 300 python tools/prof_isa.py 3 2 > gpurun_out/r2h/isa_c3_noseg.txt 2>&1
timeout 300 python tools/prof_isa.py 3 2 --no-exit > gpurun_out/r2h/isa_c3_seg_noexit.txt 2>&1
HJ_NO_SEG=1 timeout 300 python tools/prof_isa.py 3 2 --no-exit > gpurun_out/r2h/isa_c3_noseg_noexit.txt 2>&1
for f in gpurun_out/r2h/isa_c3_*.txt; do echo $f; cut -c1-250 $f; done
for k in field_coop; do timeout 300 python tools/prof_solve.py 3 f32 $k fine 1; HJ_NO_SEG=1 timeout 300 python tools/prof_solve.py 3 f32 $k fine 1; done
