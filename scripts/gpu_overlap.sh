timeout 300 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python scripts/overlap_probe.py --reps 6 --profile "FIBAR_SERIAL=0" "FIBAR_SERIAL=1" 2>&1 | cut -c1-200
