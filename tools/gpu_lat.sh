# field_lat checks + config 5 timing (usage: bash tools/gpu_lat.sh TAG)
TAG=${1:-lat}
mkdir -p gpurun_out/$TAG
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "lat or field_col or sweep_kernels_match_oracle" > gpurun_out/$TAG/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/$TAG/pytest.log
timeout 600 python tools/prof_solve.py 5 f32 auto fine 2 200 > gpurun_out/$TAG/c5_auto.txt 2>&1; tail -3 gpurun_out/$TAG/c5_auto.txt
timeout 600 python tools/prof_solve.py 5 f32 field_col fine 2 200 > gpurun_out/$TAG/c5_col.txt 2>&1; tail -3 gpurun_out/$TAG/c5_col.txt
timeout 1500 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/$TAG/bench_c5.json 2> gpurun_out/$TAG/bench.err; echo "bench c5 rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/$TAG/bench_c5.json').read().splitlines()[-1]); print(round(d['ms_per_step'],2), d['stages_ms'], 'value %.3e'%d['value'], d['roofline'].get('frac'))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d_lat --launch-skip 10 --launch-count 1 -o /tmp/c5lat python tools/prof_solve.py 5 f32 auto fine 1 20 > gpurun_out/$TAG/ncu.log 2>&1; echo "ncu rc=$?"
python tools/ncu_roofline.py /tmp/c5lat.ncu-rep c5_regulator_16385 gpurun_out/$TAG/ncu_roofline_c5_regulator_16385.json k_sweep_field2d_lat 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|dram"
python tools/ncu_sass_dump.py /tmp/c5lat.ncu-rep gpurun_out/$TAG/sass_c5lat.txt
