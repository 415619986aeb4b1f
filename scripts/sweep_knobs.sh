# Env-knob sweep on config 3 (10M-event prefix).  usage: bash scripts/sweep_knobs.sh TAG "ENV1" "ENV2" ...
TAG=$1; shift
mkdir -p gpurun_out
OUT=gpurun_out/sweep_knobs_$TAG.txt
: > $OUT
for v in "$@"; do
  line=$(env $v timeout 300 python bench.py --config 3 --events 10000000 --steps 3 --warmup 2 --no-cpu --no-e2e --no-off 2>/dev/null)
  echo "$v $(echo "$line" | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["value"],1), d["window"]["window_reruns"], d["window"]["fix_rounds"])')" | tee -a $OUT
done
