for lib in libfibar_b200.so var_noredux.so libfibar_b200.so var_noredux.so; do
  FIBAR_LIB=paper_2510_20071_b200/_lib/$lib timeout 600 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu --no-off --no-e2e > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "import json; d=json.load(open('gpurun_out/ab.json')); print('cfg3 $lib', round(d['value'],1), d['kernel_ms_per_step_serialised']['window_run'])"
done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -1
