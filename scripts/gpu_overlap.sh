timeout 300 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 600 python scripts/overlap_probe.py --reps 6 "FIBAR_SERIAL=0" 2>&1
