# A/B library builds (scratch_libs/*.so) on the micro bitmap + cfg2/cfg4 bench
for L in scratch_libs/*.so; do
  cp $L paper_1812_00282_b200/libvate_b200.so
  echo "== $L"
  python scripts/micro_bitmap.py 2>&1 | grep "kw=0"
  VARIANTS="--steps 60 --warmup 5;--config cfg4 --steps 30 --warmup 3" bash scripts/bench_variants.sh | cut -c1-140
done
