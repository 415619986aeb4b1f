# scratch runner for schedule experiments (edit freely): env knobs are read at engine creation
timeout 600 python scripts/overlap_probe.py --reps 6 "FIBAR_SERIAL=0" "FIBAR_SERIAL=1" 2>&1
