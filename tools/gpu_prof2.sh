# ncu (full, with source) of config 3's cooperative sweep and config 5's lattice sweep,
# SASS listings with per-instruction counts (usage: bash tools/gpu_prof2.sh TAG)
TAG=${1:-p2}
mkdir -p gpurun_out/$TAG
python tools/prof_step.py 3 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 5 --launch-count 1 -o /tmp/c3 python tools/prof_step.py 3 > gpurun_out/$TAG/ncu3.log 2>&1; echo "ncu3 rc=$?"
python tools/ncu_roofline.py /tmp/c3.ncu-rep c3_zermelo_4097 gpurun_out/$TAG/ncu_roofline_c3_zermelo_4097.json k_sweep_local2d_coop 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|barrier|wait"
python tools/ncu_sass_dump.py /tmp/c3.ncu-rep gpurun_out/$TAG/sass_c3.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_sweep_field2d_lat --launch-skip 10 --launch-count 1 -o /tmp/c5 python tools/prof_solve.py 5 f32 auto fine 1 20 > gpurun_out/$TAG/ncu5.log 2>&1; echo "ncu5 rc=$?"
python tools/ncu_roofline.py /tmp/c5.ncu-rep c5_regulator_16385 gpurun_out/$TAG/ncu_roofline_c5_regulator_16385.json k_sweep_field2d_lat 2>&1 | grep -E "duration|issue|warp_inst|threads_per|fma_pipe|l2_gbs|dram"
python tools/ncu_sass_dump.py /tmp/c5.ncu-rep gpurun_out/$TAG/sass_c5.txt
