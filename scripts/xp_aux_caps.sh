# aux-stream kernel CTA caps A/B: k_active (registry compaction)
V="--steps 60 --warmup 5;--config cfg3 --steps 20 --warmup 3;--config cfg4 --steps 20 --warmup 3;--config cfg1 --steps 100 --warmup 5"
for X in "VATE_XP_ACTIVE_CAP=148" "VATE_XP_ACTIVE_CAP=296" "VATE_XP_ACTIVE_CAP=444" "VATE_XP_ACTIVE_CAP=1184"; do
  echo "== $X"; env $X VARIANTS="$V" bash scripts/bench_variants.sh | cut -c1-120
done
