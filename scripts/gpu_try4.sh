mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for i in 1 2 3; do timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --no-off > gpurun_out/r2e_cfg1.json 2> gpurun_out/r2e_cfg1.err; python -c "import json; d=json.load(open('gpurun_out/r2e_cfg1.json')); print('cfg1', round(d['value'],1), round(d['e2e']['value'],1), d['config']['device_batch_cap'])"; done
