mkdir -p gpurun_out
timeout 1500 python bench.py > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/r2f_bench_reference.json 2> gpurun_out/r2f_ref.err; echo "ref rc=$?"
python -c "
import json
d=json.load(open('gpurun_out/r2f_bench.json')); r=json.load(open('gpurun_out/r2f_bench_reference.json'))
print(d['value'], d['e2e']['value'], d['parity']['frames'], d['parity']['state'], d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['traffic_ratio'], r['value'])
print({k: round(v['value']) for k, v in d['filter_off'].items()}, d['clocks'])"
