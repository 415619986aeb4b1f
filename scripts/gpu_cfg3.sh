set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
timeout 1200 python bench.py --config 3 --events 10000000 --steps 3 --warmup 3 --no-cpu > gpurun_out/cfg3.json 2> gpurun_out/cfg3.err; echo rc=$?
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu > gpurun_out/cfg1.json 2> gpurun_out/cfg1.err; echo rc=$?
