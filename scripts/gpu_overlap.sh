timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/overlap_probe.py --reps 3 --profile --w 1280 --h 720 --kind texture_noise_hot --packet 100000 "FIBAR_SERIAL=1" "FIBAR_SERIAL=0" 2>&1
