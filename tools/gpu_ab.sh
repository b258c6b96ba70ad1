# A/B of an environment switch on config 3's whole-grid and ISA fine solves
# (usage: bash tools/gpu_ab.sh TAG VAR)
TAG=${1:-ab}; VAR=${2:-HJ_COOP_GCLAIM}
mkdir -p gpurun_out/$TAG
for v in 0 1 0 1; do
  env $VAR=$v timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 > gpurun_out/$TAG/c3_$v.txt 2>&1; echo "$VAR=$v $(tail -1 gpurun_out/$TAG/c3_$v.txt)"
done
for v in 0 1; do
  env $VAR=$v timeout 600 python bench.py --config 3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c3_$v.json 2>> gpurun_out/$TAG/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c3_$v.json').read().splitlines()[-1]); print('$VAR=$v c3', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})"
done
