# aux-stream / bitmap CTA caps A/B on top of the defaults (cfg 2, cfg 3)
V="--steps 60 --warmup 5;--config cfg3 --steps 20 --warmup 3"
for X in "VATE_XP_NONE=1" "VATE_XP_BITMAP_CAP=444" "VATE_XP_BITMAP_CAP=888" "VATE_XP_INC_CAP=1184" "VATE_XP_INC_CAP=3552" "VATE_XP_FINAL_CAP=1184" "VATE_XP_NONE=1"; do
  echo "== $X"; env $X VARIANTS="$V" bash scripts/bench_variants.sh | cut -c1-110
done
