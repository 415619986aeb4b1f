# A/B of the window run's lanes per chunk (FIBAR_RUN_G small batches, FIBAR_RUN_G_LARGE large ones)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for S in "FIBAR_RUN_G=8" "FIBAR_RUN_G=4" "FIBAR_RUN_G=8 FIBAR_REG32X=0" "FIBAR_RUN_G=0"; do
  env $S timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/rung.json 2>gpurun_out/rung.err || tail -3 gpurun_out/rung.err
  python -c "import json; d=json.load(open('gpurun_out/rung.json')); k=d['kernel_ms_per_step_serialised']; print('cfg3 $S', round(d['value'],1), {n: k.get(n) for n in ('window_run','window_verify')}, d['window'])"
done
for S in "FIBAR_RUN_G_LARGE=2" "FIBAR_RUN_G_LARGE=4" "FIBAR_RUN_G_LARGE=8"; do
  env $S timeout 600 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/rung.json 2>gpurun_out/rung.err || tail -3 gpurun_out/rung.err
  python -c "import json; d=json.load(open('gpurun_out/rung.json')); k=d['kernel_ms_per_step_serialised']; print('cfg2 $S', round(d['value'],1), {n: k.get(n) for n in ('window_run','window_verify')})"
done
