#!/bin/bash
# A/B of the queue order (usage: bash tools/gpu_heavy_ab.sh TAG): HJ_COOP_HEAVY = listed-node
# threshold above which a mini-tile is queued at the front; config 3 whole grid per setting.
TAG=${1:-heavy}
mkdir -p gpurun_out/$TAG
run() {
  r=$(HJ_COOP_HEAVY=$1 HJ_COOP_QSINGLE=$2 timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 2>&1 | tail -1)
  echo "heavy=$1 qsingle=$2 :: $r" | tee -a gpurun_out/$TAG/c3_whole.txt
}
run -1 16; run 8 16; run 16 16; run 24 16; run 32 16; run 40 16; run 48 16; run 24 32; run 32 32; run 16 8; run -1 16
for c in 2 4; do for h in -1 24; do
  HJ_COOP_HEAVY=$h timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c${c}_h$h.json 2>> gpurun_out/$TAG/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c${c}_h$h.json').read().splitlines()[-1]); print('heavy=$h c$c', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})" | tee -a gpurun_out/$TAG/bench_ab.txt
done; done
