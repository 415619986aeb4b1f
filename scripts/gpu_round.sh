# Full round measurement on one B200: tests, smoke, default bench + reference arm,
# ncu launch list + full capture (gpu_full.sh), the other configs' bench lines,
# the config-4 sweep and the filter-ON halo-band emulation.
# usage: bash scripts/gpu_round.sh TAG
TAG=${1:-r1}
bash scripts/gpu_full.sh $TAG
bash scripts/gpu_configs.sh
for f in cfg1 cfg3 cfg5; do cp gpurun_out/$f.json gpurun_out/${TAG}_$f.json; done
timeout 900 python scripts/sweep_config4.py --out gpurun_out/${TAG}_config4_sweep.json 2>&1 | tail -12
timeout 900 python scripts/halo_emulate.py --config 3 --events 3000000 --bands 1,2,4,8 --halo 8 --batch 262144 --out gpurun_out/${TAG}_halo_emulate_config3_3M.json 2>&1 | tail -6
timeout 1800 python bench.py --config 3 --steps 2 --warmup 3 > gpurun_out/${TAG}_cfg3_100M.json 2> gpurun_out/${TAG}_cfg3_100M.err; echo "cfg3 100M rc=$?"
if [ -n "$FULL5" ]; then
  timeout 3000 python bench.py --config 5 --steps 2 --warmup 3 --no-cpu > gpurun_out/${TAG}_cfg5_1B.json 2> gpurun_out/${TAG}_cfg5_1B.err; echo "cfg5 1B rc=$?"
fi
