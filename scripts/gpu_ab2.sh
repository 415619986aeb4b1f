mkdir -p gpurun_out
timeout 900 python scripts/sweep_config4.py --sync --events 4000000 --max-packets 1500 --cpu-seconds 0.5 --out gpurun_out/r2d_config4_sweep_sync.json 2>&1 | grep filter | cut -c1-200
echo "== FULL_GRAPHS=1"
FIBAR_FULL_GRAPHS=1 timeout 900 python scripts/sweep_config4.py --sync --events 1000000 --max-packets 1000 --cpu-seconds 0.2 --out gpurun_out/tmp_sweep.json 2>&1 | grep '"on"' | cut -c1-200
for i in 1 2; do timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --no-off > gpurun_out/r2d_cfg1.json 2> gpurun_out/r2d_cfg1.err; python -c "import json; d=json.load(open('gpurun_out/r2d_cfg1.json')); print('cfg1', d['value'], d['e2e']['value'])"; done
