timeout 600 python -m pytest tests/test_readout.py tests/test_readout_async.py -x -q -m gpu 2>&1 | tail -4
timeout 300 python scripts/readout_bench.py 2>&1 | head -6
FIBAR_LIB=paper_2510_20071_b200/_lib/var_rot.so timeout 300 python scripts/readout_bench.py 2>&1 | tail -3
