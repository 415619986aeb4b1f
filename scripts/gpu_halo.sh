# Halo-band (filter-ON row bands) checks on one B200: GPU band tests, then the
# single-GPU emulation of 1/2/4/8 ranks on config 2 (rounds, per-rank time).
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_bands.py -q -m gpu -x 2>&1 | tail -15
timeout 1200 python scripts/halo_emulate.py --config 2 --events ${EVENTS:-3000000} --bands ${BANDS:-1,2,4,8} --halo ${HALO:-4,8} --batch ${BATCH:-262144} --out gpurun_out/halo_emulate.json 2>&1 | tail -30
