# read-out A/B: small-packet latency (config 4, 1k and 100k packets) and config 3, default build vs var_$1
V=${1:-head}
for lib in var_$V.so libfibar_b200.so; do
  echo "== $lib"
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 600 python scripts/small_packets.py 1000 300 on
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 600 python scripts/small_packets.py 1000 300 off
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 900 python bench.py --config 3 --events 5000000 --steps 3 --warmup 2 --no-cpu --no-e2e > gpurun_out/ab.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3', round(d['value'],1), d['kernel_ms_per_step'].get('sel_hist'))"
done
