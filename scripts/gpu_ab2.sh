for i in 1 2 3; do
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu --no-off > gpurun_out/cfg2.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/cfg2.json')); print('cfg2', round(d['value'],1), round(d['e2e']['value'],1), d['window'])"
done
FIBAR_TRACE=1 python scripts/cfg2_host_probe.py 2>&1 | grep -v "^[0-9]" | tail -8
