for C in 327680 458752 655360 917504; do
  timeout 600 python bench.py --config 2 --batch-cap $C --steps 5 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg2 cap $C', round(d['value'],1), d['config']['device_batch_cap'])"
done
for C in 1900544 3735552; do
  timeout 600 python bench.py --config 3 --readout end --events 30000000 --batch-cap $C --steps 3 --warmup 2 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 readout-at-end cap $C', round(d['value'],1), d['config']['device_batch_cap'])"
done
