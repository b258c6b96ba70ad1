TAG=${1:-r2u1}
mkdir -p gpurun_out/$TAG
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed|FAILED|full size" gpurun_out/$TAG/pytest_gpu.log | tail -12
timeout 1500 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c5.json 2>> gpurun_out/$TAG/bench.err; echo "bench c5 rc=$?"
timeout 900 python bench.py > gpurun_out/$TAG/bench_c3.json 2>> gpurun_out/$TAG/bench.err; echo "bench c3 rc=$?"
for c in c3 c5; do python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_$c.json').read().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), d['step_ms'], {k: round(v,2) for k,v in d['stages_ms'].items()}, 'value %.3e'%d['value'], 'frac', round(d['roofline']['frac'],4), d['labels'], d['clocks'])"; done
