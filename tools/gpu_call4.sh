#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sweep_kernels or refuses or edge_cases or stops_inside or partitioned" > gpurun_out/pytest4.log 2>&1; echo "pytest rc=$?"; tail -15 gpurun_out/pytest4.log
( for k in local_packed local_tb; do timeout 300 python tools/prof_solve.py 2 f32 $k fine 2; done
  timeout 300 python tools/prof_solve.py 2 f64 local_tb fine 1
  timeout 300 python tools/prof_solve.py 1 f64 auto fine 2 ) > gpurun_out/solve4.txt 2>&1
cat gpurun_out/solve4.txt
timeout 600 python bench.py --steps 3 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo "bench rc=$?"; cut -c1-1500 gpurun_out/bench4.json
