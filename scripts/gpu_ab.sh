# A/B of the default build against one variant (scripts/build_variants.sh NAME=...) on configs 2 and 3
V=${1:-nopf}
for lib in libfibar_b200.so var_$V.so; do
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 900 python bench.py --config 3 --events 5000000 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms_per_step']; print('$lib cfg3', round(d['value'],1), {n: k.get(n) for n in ('temporal','temporal_long','window_run')})"
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 900 python bench.py --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms_per_step']; print('$lib cfg2', round(d['value'],1), {n: k.get(n) for n in ('temporal','temporal_long','blur')})"
done
