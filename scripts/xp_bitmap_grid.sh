# bitmap-pass grid cap A/B (VATE_XP_BITMAP_CAP overrides the size rule)
echo "== rule"; VARIANTS="--steps 60 --warmup 5;--steps 60 --warmup 5;--config cfg3 --steps 20 --warmup 3;--config cfg1 --steps 100 --warmup 5;--config cfg4 --steps 20 --warmup 3" bash scripts/bench_variants.sh | cut -c1-170
for CAP in 296 444 4736; do
  echo "== cap $CAP"; VATE_XP_BITMAP_CAP=$CAP VARIANTS="--steps 60 --warmup 5;--config cfg3 --steps 20 --warmup 3;--config cfg1 --steps 100 --warmup 5" bash scripts/bench_variants.sh | cut -c1-170
done
