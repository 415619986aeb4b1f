timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 900 python scripts/overlap_probe.py --reps 5 --profile "FIBAR_GREEN=16" "FIBAR_GREEN=24" "FIBAR_GREEN=32" 2>&1 | cut -c1-230
