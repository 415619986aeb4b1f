timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 300 python scripts/packet_profile.py 1000 2>&1 | cut -c1-250
timeout 1500 python scripts/sweep_config4.py --max-packets 1500 --cpu-seconds 1 --out gpurun_out/sw3.json 2>&1 | grep -v wrote | cut -c1-140
timeout 600 python scripts/overlap_probe.py --reps 4 "FIBAR_SERIAL=0" 2>&1
