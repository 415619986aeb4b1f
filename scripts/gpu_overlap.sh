timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -1
timeout 600 python scripts/overlap_probe.py --reps 5 --profile "FIBAR_SERIAL=0" "FIBAR_SERIAL=1" 2>&1 | cut -c1-250
timeout 900 python scripts/overlap_probe.py --reps 3 --profile --w 2560 --h 1440 --events 20000000 --packet 1000000 "FIBAR_SERIAL=0" 2>&1 | cut -c1-200
