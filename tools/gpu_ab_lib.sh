#!/bin/bash
# A/B of a variant build (usage: bash tools/gpu_ab_lib.sh TAG VARIANT.so "PYTEST -k EXPR" [CONFIGS]):
# the selected GPU tests on the main libhj.so, then config 3's (and CONFIGS') whole-grid
# solve and bench line on the main build and on the variant (HJ_LIB_PATH), interleaved.
TAG=${1:-ab}; VAR=$2; KEXPR=${3:-none}; CFGS=${4:-"3"}
mkdir -p gpurun_out/$TAG
if [ "$KEXPR" != "none" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x -k "$KEXPR" > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/$TAG/pytest.log
fi
for rep in 1 2; do
for lib in main var; do
  if [ $lib = var ]; then export HJ_LIB_PATH=$PWD/$VAR; else unset HJ_LIB_PATH; fi
  timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 > gpurun_out/$TAG/c3_whole_$lib.txt 2>&1; echo "$lib c3 whole: $(tail -1 gpurun_out/$TAG/c3_whole_$lib.txt)"
  for c in $CFGS; do
    timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c${c}_$lib.json 2>> gpurun_out/$TAG/bench.err
    python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c${c}_$lib.json').read().splitlines()[-1]); print('$lib c$c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()}, d['clocks']['reasons'])"
  done
done
done
unset HJ_LIB_PATH
