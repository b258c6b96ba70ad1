mkdir -p gpurun_out
(nproc; lscpu | head -20; free -g) > gpurun_out/host_r2.txt
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2a.log 2>&1; echo smoke rc=$?
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3_r2a.json 2> gpurun_out/bench_c3_r2a.err; echo bench rc=$?
timeout 900 python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r2a.json 2> gpurun_out/bench_c5_r2a.err; echo bench5 rc=$?
