# Quick GPU check (usage: bash tools/gpu_quick.sh TAG "PYTEST -k EXPR" "BENCH CONFIGS"):
# a pytest selection, whole-grid timings of configs 3 and 5, bench lines.
TAG=${1:-q}; KEXPR=${2:-lat}; CFGS=${3:-"3"}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$TAG/build.log 2>&1
if [ "$KEXPR" != "none" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -k "$KEXPR" > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/$TAG/pytest.log
fi
timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 > gpurun_out/$TAG/c3_whole.txt 2>&1; tail -1 gpurun_out/$TAG/c3_whole.txt
timeout 300 python tools/prof_solve.py 5 f32 auto fine 2 200 > gpurun_out/$TAG/c5_200.txt 2>&1; tail -1 gpurun_out/$TAG/c5_200.txt
for c in $CFGS; do
  S=5; [ "$c" = "5" ] && S=1
  timeout 1500 python bench.py --config $c --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c$c.json 2>> gpurun_out/$TAG/bench.err; echo "bench c$c rc=$?"
  python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c$c.json').read().splitlines()[-1]); print('c$c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()}, 'value %.3e'%d['value'], 'frac', round(d['roofline']['frac'],4), d['clocks']['reasons'])"
done
