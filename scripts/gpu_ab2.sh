timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python scripts/sweep_config4.py --sync --events 4000000 --max-packets 1500 --cpu-seconds 0.3 --out gpurun_out/r2e_config4_sweep_sync.json 2>&1 | grep '"packet": 1000,' | cut -c1-170
timeout 900 python scripts/sweep_config4.py --events 20000000 --out gpurun_out/r2e_config4_sweep.json 2>&1 | grep '"packet": 1000,' | cut -c1-170
