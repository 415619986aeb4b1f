# config 3 (per-packet read-out) under read-out scheduling knobs
for v in 32768 -1 131072; do
  echo "== FIBAR_ASYNC_GRAPH_MAX=$v"
  FIBAR_ASYNC_GRAPH_MAX=$v timeout 900 python bench.py --config 3 --events 5000000 --steps 3 --warmup 2 --no-cpu > gpurun_out/c3o.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/c3o.json')); print(round(d['value'],1), round(d['e2e']['value'],1))"
done
