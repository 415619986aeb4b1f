timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" 2>&1 | tail -1
timeout 900 python scripts/overlap_probe.py --reps 5 "FIBAR_GREEN=16" "FIBAR_GREEN=0" 2>&1 | cut -c1-130
