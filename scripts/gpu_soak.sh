# repeat the GPU suite and smoke to catch anything flaky
for i in 1 2 3 4 5 6; do timeout 900 python -m pytest tests -q -m gpu -x -p no:cacheprovider 2>&1 | tail -1; done
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for i in 1 2; do timeout 900 python bench.py --config 3 --events 20000000 --steps 3 --warmup 3 --no-off > gpurun_out/soak.json 2> gpurun_out/soak.err; python -c "import json; d=json.load(open('gpurun_out/soak.json')); print('cfg3 20M', round(d['value'],1), round(d['e2e']['value'],1), d['parity']['frames'], d['parity']['state'], d['roofline']['traffic'])"; done
