mkdir -p gpurun_out/c4band
for b in 4 8 16; do
timeout 600 python tools/diag_isa_gap.py 4 1.0 exit $b > gpurun_out/c4band/diag_c4_band$b.txt 2>&1; echo "diag c4 band $b rc=$?"; head -4 gpurun_out/c4band/diag_c4_band$b.txt
done
timeout 600 python tools/prof_isa.py 5 1 --shares > gpurun_out/c4band/shares_c5.txt 2>&1; tail -5 gpurun_out/c4band/shares_c5.txt
timeout 600 python tools/prof_isa.py 3 1 --shares > gpurun_out/c4band/shares_c3.txt 2>&1; tail -5 gpurun_out/c4band/shares_c3.txt
for rep in 1 2; do for lib in main var; do
  if [ $lib = var ]; then export HJ_LIB_PATH=$PWD/paper_1405_3521_b200/_lib/var_nw8.so; else unset HJ_LIB_PATH; fi
  timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4band/bench_c4_$lib.json 2>> gpurun_out/c4band/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/c4band/bench_c4_$lib.json').read().splitlines()[-1]); print('$lib c4', round(d['ms_per_step'],2), {k: round(v,2) for k,v in d['stages_ms'].items()})"
  timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/c4band/bench_c1_$lib.json 2>> gpurun_out/c4band/bench.err
  python -c "
import json; d=json.loads(open('gpurun_out/c4band/bench_c1_$lib.json').read().splitlines()[-1]); print('$lib c1', round(d['ms_per_step'],3), {k: round(v,2) for k,v in d['stages_ms'].items()})"
done; done
unset HJ_LIB_PATH
