for S in "FIBAR_SORT_LANES=2" "FIBAR_SORT_LANES=3" "FIBAR_SORT_LANES=2 FIBAR_LIB=paper_2510_20071_b200/_lib/var_npar7.so" "FIBAR_SORT_LANES=3 FIBAR_LIB=paper_2510_20071_b200/_lib/var_npar7.so"; do
  env $S timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 $S', round(d['value'],1), round(d['e2e']['value'],1))"
done
