# Window speculation warm-up on config 3 (10M-event prefix, per-packet read-out).
# usage: bash scripts/sweep_window.sh TAG [warms...]
TAG=${1:-r2}
shift
WARMS=${@:-64 48 32 24}
mkdir -p gpurun_out
OUT=gpurun_out/sweep_window_$TAG.txt
: > $OUT
for w in $WARMS; do
  line=$(FIBAR_WARM=$w timeout 300 python bench.py --config 3 --events 10000000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-off 2>/dev/null)
  echo "warm=$w $(echo "$line" | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],1), d["window"], {k: v for k, v in list(d["kernel_ms_per_step_serialised"].items())[:10]})')" | tee -a $OUT
done
