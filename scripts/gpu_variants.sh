# Scratch: compare library variants (scripts/build_variants.sh) on config 2 and a config-3 prefix.
# usage: bash scripts/gpu_variants.sh base pf2 pf4 ...   (base = the default build)
L=paper_2510_20071_b200/_lib
for v in "$@"; do
  lib=$L/libfibar_b200.so; [ "$v" != base ] && lib=$L/var_$v.so
  echo "== $v"
  FIBAR_LIB=$lib timeout 600 python scripts/overlap_probe.py --reps 5 ${SETTINGS:-"FIBAR_GREEN=16"} 2>&1 | cut -c1-200
  FIBAR_LIB=$lib timeout 600 python scripts/overlap_probe.py --reps 3 --w 1280 --h 720 --kind texture_noise_hot --packet 100000 "FIBAR_GREEN=16" 2>&1 | cut -c1-200
done
