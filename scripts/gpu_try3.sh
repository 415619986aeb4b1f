mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-off > gpurun_out/cfg2.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/cfg2.json')); k=d['kernel_ms_per_step_serialised']; print('cfg2', round(d['value'],1), round(d['e2e']['value'],1), {n:k.get(n) for n in ('rs_scatter','rs_hist','scan','scan_apply','scan_reduce')})"
timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms_per_step_serialised']; print('cfg3', round(d['value'],1), round(d['e2e']['value'],1), {n:k.get(n) for n in ('rs_scatter','rs_hist','scan')})"
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); k=d['kernel_ms_per_step_serialised']; print('cfg1', round(d['value'],1), round(d['e2e']['value'],1), k)"
timeout 600 python bench.py --config 5 --events 30000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg5', round(d['value'],1))"
