mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/try.json 2>gpurun_out/try.err || tail -3 gpurun_out/try.err
python -c "import json; d=json.load(open('gpurun_out/try.json')); k=d['kernel_ms_per_step_serialised']; print('cfg3', round(d['value'],1), k)"
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/try.json 2>gpurun_out/try.err || tail -3 gpurun_out/try.err
python -c "import json; d=json.load(open('gpurun_out/try.json')); print('cfg2', round(d['value'],1))"
TRACE_ROWS=1 timeout 300 python scripts/trace_parts.py 6000000 2>&1 | tail -18
