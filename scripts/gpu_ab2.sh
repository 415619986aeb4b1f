timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --no-off > gpurun_out/r2e_cfg1.json 2> gpurun_out/r2e_cfg1.err; python -c "import json; d=json.load(open('gpurun_out/r2e_cfg1.json')); print('cfg1', round(d['value'],1), round(d['e2e']['value'],1), d['parity']['state'], d['gpu_launches'])"; done
timeout 900 python scripts/sweep_config4.py --sync --events 4000000 --max-packets 1500 --cpu-seconds 0.3 --out gpurun_out/tmp_sync.json 2>&1 | grep '"off"' | cut -c1-170
timeout 900 python scripts/sweep_config4.py --events 20000000 --cpu-seconds 0.3 --out gpurun_out/tmp_async.json 2>&1 | grep '"off"' | cut -c1-170
