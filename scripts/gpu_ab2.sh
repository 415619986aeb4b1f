for S in "FIBAR_ANCHOR_STREAM=0" "FIBAR_ANCHOR_STREAM=1" "FIBAR_ANCHOR_STREAM=0" "FIBAR_ANCHOR_STREAM=1"; do
  env $S timeout 600 python bench.py --config 3 --events 20000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 20M $S', round(d['value'],1), round(d['e2e']['value'],1))"
done
FIBAR_ANCHOR_STREAM=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "small_packets or schedule_knobs or graph" 2>&1 | tail -2
