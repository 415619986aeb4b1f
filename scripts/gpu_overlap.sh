timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/overlap_probe.py --reps 4 --profile "FIBAR_SERIAL=1" "FIBAR_SERIAL=0" "FIBAR_BLUR_BLOCKS=2" 2>&1
