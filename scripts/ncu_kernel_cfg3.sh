# ncu --set full of chosen kernels on config 3 in steady state (skips the first
# launches of those kernels).  usage: bash scripts/ncu_kernel_cfg3.sh TAG REGEX [SKIP] [COUNT] [ENV...]
TAG=$1; RE=$2; SKIP=${3:-40}; CNT=${4:-2}
shift 4
mkdir -p gpurun_out
ARGS="--config 3 --profile-only --events 6000000"
env "$@" python bench.py $ARGS > gpurun_out/plainK_$TAG.log 2>&1 && \
env FIBAR_GREEN=0 "$@" ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT -o gpurun_out/fullK_$TAG python bench.py $ARGS > gpurun_out/ncuK_$TAG.log 2>&1
echo "ncu rc=$?"
