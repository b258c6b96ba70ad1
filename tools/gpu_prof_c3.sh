mkdir -p gpurun_out/p1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python tools/coop_trace.py 3 isa > gpurun_out/p1/trace_c3_isa.txt 2>&1
python tools/coop_trace.py 3 > gpurun_out/p1/trace_c3_whole.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep_local2d_coop --launch-skip 5 --launch-count 1 -o /tmp/c3 python tools/prof_step.py 3 > gpurun_out/p1/ncu.log 2>&1
python tools/ncu_sass_dump.py /tmp/c3.ncu-rep gpurun_out/p1/sass_c3.txt
ncu -i /tmp/c3.ncu-rep --page raw --csv > gpurun_out/p1/raw_c3.csv 2>&1
ls -la gpurun_out/p1
