for i in 1 2 3; do
timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3', round(d['value'],1), round(d['e2e']['value'],1))"
done
python scripts/e2e_profile.py 2>&1 | grep "run()"
