set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
ARGS="--profile-only --events 3145728 --batch-cap 1048576"
python bench.py $ARGS > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_blur$|k_window_run|k_anchor$" -s 3 -c 3 -o gpurun_out/prof_$1 python bench.py $ARGS > gpurun_out/ncu_$1.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/ncu_$1.log
