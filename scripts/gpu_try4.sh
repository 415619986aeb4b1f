mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-off > gpurun_out/r2e_cfg2.json 2> gpurun_out/r2e_cfg2.err; echo "cfg2 rc=$?"
timeout 1500 python bench.py --config 5 --events 30000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/r2e_cfg5.json 2> gpurun_out/r2e_cfg5.err; echo "cfg5 rc=$?"
python -c "
import json
for f in ('r2e_cfg2','r2e_cfg5'):
    d=json.load(open('gpurun_out/'+f+'.json')); print(f, round(d['value'],1), round(d['e2e']['value'],1), (d.get('parity') or {}).get('state'))"
timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 10M', round(d['value'],1), round(d['e2e']['value'],1))"
