for P in 0.05 0.05 0.05 0.05 1000 1000 1000 1000; do
  BENCH_CLOCK_PERIOD=$P timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg2 period $P', round(d['value'],1), d['clocks']['samples'])"
done
for P in 0.05 1000 0.05 1000; do
  BENCH_CLOCK_PERIOD=$P timeout 600 python bench.py --config 3 --events 20000000 --steps 5 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 period $P', round(d['value'],1), d['clocks']['samples'])"
done
