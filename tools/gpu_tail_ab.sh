#!/bin/bash
# A/B of the cooperative sweep's load-balance switches on config 3 (usage: bash
# tools/gpu_tail_ab.sh TAG): the whole-grid solve (prof_solve, 2 reps, last line kept) per
# setting of HJ_COOP_TAIL (16ths of the list claimed dynamically), HJ_COOP_TCH (chunk) and
# HJ_COOP_QSINGLE (single-item claims at the end of a CTA's queue); then bit-identity of the
# best against the default and bench lines.
TAG=${1:-tail}
mkdir -p gpurun_out/$TAG
run() {  # TAIL TCH QSINGLE
  r=$(HJ_COOP_TAIL=$1 HJ_COOP_TCH=$2 HJ_COOP_QSINGLE=$3 timeout 300 python tools/prof_solve.py 3 f32 auto fine 2 2>&1 | tail -1)
  echo "tail=$1 tch=$2 qsingle=$3 :: $r" | tee -a gpurun_out/$TAG/c3_whole.txt
}
run 0 32 0
run 0 32 16
run 0 32 32
run 4 32 0
run 8 32 0
run 12 32 0
run 16 32 0
run 8 64 0
run 8 16 0
run 8 32 16
run 12 32 16
run 12 16 16
run 0 32 0
