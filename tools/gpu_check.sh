#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (default + every config), ncu launch list.
# Usage (from the repo root, on the GPU box):  bash tools/gpu_check.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$tag.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_$tag.log
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv -lms 200 > gpurun_out/clocks_$tag.csv &
SMI=$!
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
for c in 1 3 4; do
  timeout 900 python bench.py --config $c --steps 2 --no-cpu-baseline > gpurun_out/bench_c${c}_$tag.json 2>> gpurun_out/bench_$tag.err; echo "bench c$c rc=$?"
done
kill $SMI
cat gpurun_out/bench_*_$tag.json gpurun_out/bench_$tag.json | cut -c1-400
# launch list of one bench step (cold-cache, serialised; compare shares)
python tools/prof_step.py 2 > gpurun_out/prof_plain_$tag.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv \
    --log-file gpurun_out/launches_$tag.csv python tools/prof_step.py 2 > gpurun_out/ncu_launch_$tag.log 2>&1
echo "ncu rc=$?"
python tools/launch_stats.py gpurun_out/launches_$tag.csv | head -20
# the largest config (16385^2, 32 sub-domains): one timed step after the required warm-ups
if [ "${WITH_C5:-0}" = "1" ]; then
  timeout 2400 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$tag.json 2>> gpurun_out/bench_$tag.err; echo "bench c5 rc=$?"
  cut -c1-600 gpurun_out/bench_c5_$tag.json
fi
