timeout 300 python -m pytest tests -x -q -m gpu 2>&1 | tail -2
timeout 600 python scripts/overlap_probe.py --reps 6 "FIBAR_PDL=1" "FIBAR_PDL=0" "FIBAR_PDL=1 FIBAR_SERIAL=1" "FIBAR_PDL=0 FIBAR_SERIAL=1" 2>&1
timeout 1500 python scripts/sweep_config4.py --max-packets 1500 --cpu-seconds 1 --out gpurun_out/sw4.json 2>&1 | grep -v wrote | cut -c1-140
FIBAR_PDL=0 timeout 1500 python scripts/sweep_config4.py --max-packets 1500 --cpu-seconds 1 --out gpurun_out/sw4n.json 2>&1 | grep -v wrote | cut -c1-140
