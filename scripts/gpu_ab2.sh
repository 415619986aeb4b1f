mkdir -p gpurun_out
for S in "FIBAR_LIB=paper_2510_20071_b200/_lib/var_npar7.so" "FIBAR_LIB=paper_2510_20071_b200/_lib/var_npar10.so"; do
  env $S timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 $S', round(d['value'],1))"
  env $S TRACE_ROWS=1 timeout 300 python scripts/trace_parts.py 6000000 2>&1 | tail -18 | head -9
done
