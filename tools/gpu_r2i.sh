#!/bin/bash
# full GPU suite, smoke, bench (default config 3) + config 2/4/5 lines, ncu of the config-3 fine launch
mkdir -p gpurun_out/r2i
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2i/smoke.log 2>&1; echo "smoke rc=$?"
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2i/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -50 gpurun_out/r2i/pytest_gpu.log
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/r2i/clocks.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/r2i/bench_c3.json 2> gpurun_out/r2i/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2i/bench_c2.json 2>> gpurun_out/r2i/bench.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/r2i/bench_c4.json 2>> gpurun_out/r2i/bench.err; echo "bench c4 rc=$?"
timeout 600 python bench.py --config 1 --no-cpu-baseline > gpurun_out/r2i/bench_c1.json 2>> gpurun_out/r2i/bench.err; echo "bench c1 rc=$?"
timeout 1500 python bench.py --config 5 --steps 1 --no-cpu-baseline > gpurun_out/r2i/bench_c5.json 2>> gpurun_out/r2i/bench.err; echo "bench c5 rc=$?"
kill $SMI
for c in c3 c2 c4 c1 c5; do python -c "
import json; d=json.loads(open('gpurun_out/r2i/bench_$c.json').read().splitlines()[-1]); print('$c', round(d['ms_per_step'],2), d['stages_ms'], 'frac', round(d['roofline']['frac'],4), d['labels'], d['clocks'])"; done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r2i/bench_ref.json 2>> gpurun_out/r2i/bench.err; echo "ref rc=$?"; cut -c1-300 gpurun_out/r2i/bench_ref.json
python tools/prof_step.py 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/r2i/launches_c3_step.csv python tools/prof_step.py 3 > gpurun_out/r2i/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_stats.py gpurun_out/r2i/launches_c3_step.csv > gpurun_out/r2i/launches_c3_step.txt 2>&1; head -14 gpurun_out/r2i/launches_c3_step.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 5 --launch-count 1 \
    -o gpurun_out/r2i/ncu_c3_fine python tools/prof_step.py 3 > gpurun_out/r2i/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_roofline.py gpurun_out/r2i/ncu_c3_fine.ncu-rep c3_zermelo_4097 gpurun_out/r2i/ncu_roofline_c3_zermelo_4097.json k_sweep_local2d_coop 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|barrier|wait"
