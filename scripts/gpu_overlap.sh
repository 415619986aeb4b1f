timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -1
timeout 900 python scripts/overlap_probe.py --reps 5 --profile "FIBAR_GREEN=16" "FIBAR_SERIAL=1" 2>&1 | cut -c1-230
timeout 900 python scripts/overlap_probe.py --reps 3 --w 1280 --h 720 --kind texture_noise_hot --packet 100000 "FIBAR_GREEN=16" 2>&1 | cut -c1-120
