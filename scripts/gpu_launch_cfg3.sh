# ncu launch list + --set full of the top window kernels on config 3 in steady
# state: a 6M-event prefix (60 packets of 100k, per-packet read-out), skipping
# the first 40 packets' launches (the window takes ~4 packets to fill and the
# first captured graphs), then 20 packets.
# usage: bash scripts/gpu_launch_cfg3.sh TAG [skip_launches]
TAG=${1:-r2}
SKIP=${2:-1400}
mkdir -p gpurun_out
ARGS="--config 3 --profile-only --events 6000000"
python bench.py $ARGS > gpurun_out/plain_c3_$TAG.log 2>&1 && \
FIBAR_GREEN=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv -s $SKIP -c 700 --log-file gpurun_out/launches_c3_$TAG.csv python bench.py $ARGS > gpurun_out/ncu_launch_c3_$TAG.log 2>&1
echo "launch list rc=$?"
python scripts/launch_table.py gpurun_out/launches_c3_$TAG.csv 20 | head -40
if [ -n "$FULL" ]; then
FIBAR_GREEN=0 ncu --set full --clock-control none --import-source on -k regex:"$FULL" -s 40 -c 3 -o gpurun_out/full_c3_$TAG python bench.py $ARGS > gpurun_out/ncu_full_c3_$TAG.log 2>&1
echo "ncu full rc=$?"
fi
