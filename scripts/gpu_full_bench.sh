mkdir -p gpurun_out
TAG=${1:-r2c}
timeout 1700 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/${TAG}_bench.err
python -c "
import json; d=json.load(open('gpurun_out/${TAG}_bench.json'))
print(d['value'], d['e2e']['value'], d['parity'], d['roofline']['kernel'], d['roofline']['frac'], d['cpu_baseline']['value'])
print(d['filter_off'])"
