# Round measurement: tests, smoke, bench, ncu launch list, ncu full capture of the top kernels.
# usage: bash scripts/gpu_full.sh TAG
set -x
TAG=${1:-r1}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2>&1; echo "ref rc=$?"
ARGS="--profile-only --events 3145728"
# (the launch list runs without the blur's green-context partition: ncu cannot
# replay every kernel of a step inside a green context; the kernels are the same)
python bench.py $ARGS > gpurun_out/plain_$TAG.log 2>&1 && \
FIBAR_GREEN=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_$TAG.log 2>&1
echo "launch list rc=$?"
python bench.py $ARGS > gpurun_out/plain2_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_blur$|k_window_run|k_anchor$|k_rs_scatter" -s 2 -c 4 -o gpurun_out/full_$TAG python bench.py $ARGS > gpurun_out/ncu_full_$TAG.log 2>&1
echo "ncu full rc=$?"
cat gpurun_out/bench_$TAG.json; cat gpurun_out/bench_ref_$TAG.json
