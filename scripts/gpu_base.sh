# Baseline on one B200: GPU tests, smoke, config-3 full-stream bench line.
# usage: bash scripts/gpu_base.sh TAG
TAG=${1:-r2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
( time timeout 1800 python bench.py --config 3 --steps 2 --warmup 3 ) > gpurun_out/${TAG}_cfg3_100M.json 2> gpurun_out/${TAG}_cfg3_100M.err; echo "cfg3 rc=$?"
tail -5 gpurun_out/${TAG}_cfg3_100M.err
