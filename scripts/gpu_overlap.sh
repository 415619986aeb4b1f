timeout 300 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/overlap_probe.py --reps 6 "FIBAR_SERIAL=0" "FIBAR_SERIAL=1" "FIBAR_BLUR_BLOCKS=1" "FIBAR_BLUR_BLOCKS=2" "FIBAR_SERIAL=0" 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>&1 | cut -c1-400
