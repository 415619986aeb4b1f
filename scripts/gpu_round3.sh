# Round-2 (second half) measurement set on one B200: tests, smoke, the default
# bench (config 3 full stream) + reference arm, the ncu launch list and a
# --set full capture of the step's top kernels on a config-3 prefix, the other
# configs' lines, the config-4 sweep and the stream-part timeline.
# usage: bash scripts/gpu_round3.sh TAG
TAG=${1:-r2e}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 1 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
ARGS="--config 3 --profile-only --events 6000000"
python bench.py $ARGS > gpurun_out/${TAG}_plain.log 2>&1; tail -1 gpurun_out/${TAG}_plain.log > gpurun_out/${TAG}_profile_meta.json
# steady state: skip the first 1200 launches (the window fills over ~4 packets), then 1000 launches
ncu --metrics gpu__time_duration.sum --clock-control none --csv -s 1200 -c 1000 --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launch list rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_window_run|k_window_verify|k_anchor2|k_readout|k_rs_scatter|k_blur_prep|k_temporal_long" -s 70 -c 7 -o gpurun_out/full_${TAG} python bench.py $ARGS > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "ncu full rc=$?"
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-off > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err; echo "cfg2 rc=$?"
timeout 900 python bench.py --config 1 --steps 5 --warmup 3 --no-off > gpurun_out/${TAG}_cfg1.json 2> gpurun_out/${TAG}_cfg1.err; echo "cfg1 rc=$?"
timeout 1500 python bench.py --config 5 --events 30000000 --steps 3 --warmup 3 --no-cpu --no-off > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err; echo "cfg5 rc=$?"
timeout 900 python scripts/sweep_config4.py --out gpurun_out/${TAG}_config4_sweep.json 2>&1 | tail -10
TRACE_ROWS=1 timeout 300 python scripts/trace_parts.py 6000000 > gpurun_out/${TAG}_trace_parts.txt 2>&1
cat gpurun_out/${TAG}_trace_parts.txt
timeout 900 python scripts/sweep_config4.py --sync --events 4000000 --max-packets 1500 --cpu-seconds 0.5 --out gpurun_out/${TAG}_config4_sweep_sync.json 2>&1 | tail -8 | cut -c1-160
