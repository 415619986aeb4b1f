for i in 1 2 3; do timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r2g_bench.json 2> gpurun_out/r2g_bench.err; echo "bench rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r2g_bench.json'))
print(d['value'], d['e2e']['value'], d['parity']['frames'], d['parity']['state'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic_ratio'], d['cpu_baseline']['value'], d['gpu_launches'])
print({k: round(v['value']) for k, v in d['filter_off'].items()}, d['clocks'])"
