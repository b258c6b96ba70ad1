#!/bin/bash
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()"
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest10.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest10.log
( timeout 300 python tools/prof_solve.py 2 f32 local_tb fine 2
  timeout 300 python tools/prof_solve.py 2 f32 local_packed fine 1
  timeout 300 python tools/prof_solve.py 2 f32 local_tb coarse 2
  timeout 300 python tools/prof_solve.py 3 f32 auto fine 1
  timeout 300 python tools/prof_solve.py 4 f32 auto fine 2
  timeout 300 python tools/prof_solve.py 1 f64 auto fine 2 ) > gpurun_out/solve10.txt 2>&1
cat gpurun_out/solve10.txt
timeout 600 python bench.py --steps 3 > gpurun_out/bench10.json 2> gpurun_out/bench10.err; echo "bench rc=$?"
timeout 600 python bench.py --config 4 --steps 2 --no-cpu-baseline > gpurun_out/bench10_c4.json 2>> gpurun_out/bench10.err
timeout 900 python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench10_c3.json 2>> gpurun_out/bench10.err
python - <<'PY'
import json
for f in ['bench10.json','bench10_c4.json','bench10_c3.json']:
    try:
        d=json.loads(open('gpurun_out/'+f).read().strip().splitlines()[-1])
        print(f, round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()}, d['fine_sweeps'], 'frac', round(d['roofline']['frac'],4))
    except Exception as e: print(f, e)
PY
