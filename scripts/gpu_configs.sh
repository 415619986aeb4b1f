# bench lines for the other BASELINE configs (informational, profiles/)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/cfg2.json 2> gpurun_out/cfg2.err; echo rc=$?
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/cfg1.json 2> gpurun_out/cfg1.err; echo rc=$?
timeout 1200 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo rc=$?
tail -3 gpurun_out/cfg3.err
timeout 1500 python bench.py --config 5 --events 30000000 --steps 3 --warmup 3 --no-cpu > gpurun_out/cfg5.json 2> gpurun_out/cfg5.err; echo rc=$?
tail -3 gpurun_out/cfg5.err
for f in cfg2 cfg1 cfg3 cfg5; do python -c "
import json; d = json.load(open('gpurun_out/$f.json'))
print('$f', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1) if d.get('e2e') else None, 'cpu', round((d.get('cpu_baseline') or {}).get('value',0),1), 'ms/step', round(d['ms_per_step'],2))
print('   kernels', {k: v for k, v in list(d['kernel_ms_per_step'].items())[:8]})
print('   window', d.get('window'))
"; done
