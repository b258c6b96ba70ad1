#!/bin/bash
# round 2, call b: smoke, full GPU suite, bench (default config 3 + config 2), ncu evidence
mkdir -p gpurun_out/r2b
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r2b/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r2b/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/r2b/bench_c3.json 2> gpurun_out/r2b/bench_c3.err; echo "bench rc=$?"
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/r2b/bench_c2.json 2>> gpurun_out/r2b/bench_c3.err; echo "bench c2 rc=$?"
timeout 600 python bench.py --config 4 --steps 2 --no-cpu-baseline > gpurun_out/r2b/bench_c4.json 2>> gpurun_out/r2b/bench_c3.err; echo "bench c4 rc=$?"
cut -c1-1500 gpurun_out/r2b/bench_c3.json
python tools/prof_step.py 3 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/r2b/launches_c3_step.csv python tools/prof_step.py 3 > gpurun_out/r2b/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/launch_stats.py gpurun_out/r2b/launches_c3_step.csv > gpurun_out/r2b/launches_c3_step.txt 2>&1; head -20 gpurun_out/r2b/launches_c3_step.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 3 --launch-count 1 \
    -o gpurun_out/r2b/ncu_c3_fine python tools/prof_step.py 3 > gpurun_out/r2b/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/ncu_roofline.py gpurun_out/r2b/ncu_c3_fine.ncu-rep c3_zermelo_4097 gpurun_out/r2b/ncu_roofline_c3_zermelo_4097.json k_sweep_local2d_coop > /dev/null 2>&1; echo "summary rc=$?"
