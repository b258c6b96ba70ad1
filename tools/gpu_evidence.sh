#!/bin/bash
# One evidence run on the GPU box (usage: bash tools/gpu_evidence.sh TAG): smoke, the full
# GPU suite, bench lines (default config 3, configs 1/2/4/5), the reference arm, the launch
# list of a config-3 step and ncu summaries of the config-3 and config-5 sweep kernels, all
# under gpurun_out/TAG (ncu reports stay on the box: gpurun_out comes back capped at 64 MiB).
TAG=${1:-r2t}
mkdir -p gpurun_out/$TAG
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/$TAG/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/$TAG/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -45 gpurun_out/$TAG/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/$TAG/bench_c3.json 2> gpurun_out/$TAG/bench.err; echo "bench rc=$?"
for c in 1 2 4; do timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/$TAG/bench_c$c.json 2>> gpurun_out/$TAG/bench.err; echo "bench c$c rc=$?"; done
timeout 1500 python bench.py --config 5 --steps 1 --no-cpu-baseline > gpurun_out/$TAG/bench_c5.json 2>> gpurun_out/$TAG/bench.err; echo "bench c5 rc=$?"
for c in c3 c1 c2 c4 c5; do python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_$c.json').read().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), d['step_ms'], {k: round(v,2) for k,v in d['stages_ms'].items()}, 'value %.3e'%d['value'], 'frac', round(d['roofline']['frac'],4), 'e2e ms', round(d['e2e']['ms_per_step'],2), d['clocks'])"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/$TAG/bench_ref.json 2>> gpurun_out/$TAG/bench.err; echo "ref rc=$?"
python tools/prof_step.py 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/$TAG/launches_c3_step.csv python tools/prof_step.py 3 > gpurun_out/$TAG/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_stats.py gpurun_out/$TAG/launches_c3_step.csv > gpurun_out/$TAG/launches_c3_step.txt 2>&1; head -14 gpurun_out/$TAG/launches_c3_step.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 5 --launch-count 1 \
    -o gpurun_out/$TAG/ncu_c3_fine python tools/prof_step.py 3 > gpurun_out/$TAG/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_roofline.py gpurun_out/$TAG/ncu_c3_fine.ncu-rep c3_zermelo_4097 gpurun_out/$TAG/ncu_roofline_c3_zermelo_4097.json k_sweep_local2d_coop 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|barrier|wait"
python tools/ncu_source.py gpurun_out/$TAG/ncu_c3_fine.ncu-rep 40 > gpurun_out/$TAG/ncu_c3_fine_hotspots.txt 2>&1
python tools/ncu_summary.py gpurun_out/$TAG/ncu_c3_fine.ncu-rep > gpurun_out/$TAG/ncu_c3_fine_summary.txt 2>&1
python tools/ncu_sass_dump.py gpurun_out/$TAG/ncu_c3_fine.ncu-rep gpurun_out/$TAG/sass_c3.txt
mv gpurun_out/$TAG/ncu_c3_fine.ncu-rep /tmp/   # (reports stay on the box: gpurun_out is capped at 64 MiB)
python tools/prof_solve.py 5 f32 auto fine 1 20 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d_lat --launch-skip 10 --launch-count 1 \
    -o gpurun_out/$TAG/ncu_c5_col python tools/prof_solve.py 5 f32 auto fine 1 20 > gpurun_out/$TAG/ncu5.log 2>&1; echo "ncu c5 rc=$?"
python tools/ncu_roofline.py gpurun_out/$TAG/ncu_c5_col.ncu-rep c5_regulator_16385 gpurun_out/$TAG/ncu_roofline_c5_regulator_16385.json k_sweep_field2d_lat > /dev/null 2>&1
python tools/ncu_source.py gpurun_out/$TAG/ncu_c5_col.ncu-rep 40 > gpurun_out/$TAG/ncu_c5_col_hotspots.txt 2>&1
mv gpurun_out/$TAG/ncu_c5_col.ncu-rep /tmp/
du -sh gpurun_out/$TAG
