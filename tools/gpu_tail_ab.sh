#!/bin/bash
# A/B of the cooperative sweep's intra-CTA balance switch (usage: bash tools/gpu_tail_ab.sh
# TAG): HJ_COOP_QSINGLE = how many items at the end of a CTA's queue are claimed one at a
# time; config 3's whole-grid solve per setting (prof_solve, 2 reps, last line kept), then
# bench lines of configs 3, 2 and 4 with pairs only (0) and the default.
TAG=${1:-tail}
mkdir -p gpurun_out/$TAG
run() {
  r=$(HJ_COOP_QSINGLE=$1 timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 2>&1 | tail -1)
  echo "qsingle=$1 :: $r" | tee -a gpurun_out/$TAG/c3_whole.txt
}
for q in 0 8 16 24 32 48 100000 0 16; do run $q; done
for c in 3 2 4; do for q in 0 default; do
  if [ $q = default ]; then unset HJ_COOP_QSINGLE; else export HJ_COOP_QSINGLE=$q; fi
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c${c}_q$q.json 2>> gpurun_out/$TAG/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c${c}_q$q.json').read().splitlines()[-1]); print('qsingle=$q c$c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})" | tee -a gpurun_out/$TAG/bench_ab.txt
done; done
