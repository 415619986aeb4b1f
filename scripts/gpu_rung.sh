# A/B of window-run settings
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for S in "FIBAR_RUN_G=8" "FIBAR_RUN_G=4" "FIBAR_RUN_G=8 FIBAR_WARM=16" "FIBAR_RUN_G=8 FIBAR_WARM=24"; do
  env $S timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/rung.json 2>gpurun_out/rung.err || tail -3 gpurun_out/rung.err
  python -c "import json; d=json.load(open('gpurun_out/rung.json')); k=d['kernel_ms_per_step_serialised']; print('cfg3 $S', round(d['value'],1), {n: k.get(n) for n in ('window_run','window_verify','temporal','temporal_long')}, d['window']['window_reruns'], d['window']['fix_rounds'])"
done
for S in "FIBAR_RUN_G_LARGE=4" "FIBAR_RUN_G_LARGE=8"; do
  env $S timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/rung.json 2>gpurun_out/rung.err || tail -3 gpurun_out/rung.err
  python -c "import json; d=json.load(open('gpurun_out/rung.json')); k=d['kernel_ms_per_step_serialised']; print('cfg2 $S', round(d['value'],1), {n: k.get(n) for n in ('window_run','window_verify','temporal','temporal_long')})"
done
timeout 300 python scripts/trace_parts.py 6000000 2>&1 | tail -12
