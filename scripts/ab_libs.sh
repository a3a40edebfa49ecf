# A/B library builds (scratch_libs/*.so): cfg2 / cfg3 bench
for L in scratch_libs/*.so; do
  cp $L paper_1812_00282_b200/libvate_b200.so
  echo "== $L"
  VARIANTS="${AB_VARIANTS:---steps 60 --warmup 5;--config cfg3 --steps 30 --warmup 3}" bash scripts/bench_variants.sh | cut -c1-150
done
