# bench variants: args per line in $VARIANTS (";"-separated); prints a compact summary per run
IFS=';'
for V in $VARIANTS; do
  unset IFS
  python bench.py $V > gpurun_out/variant.json 2>/dev/null
  python - "$V" <<'PY'
import json, sys
try:
    d = json.loads(open("gpurun_out/variant.json").read().strip().splitlines()[-1])
except Exception as e:
    print(sys.argv[1], "FAILED", e); sys.exit()
print(sys.argv[1], "|", d["config"]["workload"], "value", round(d["value"]), "ms", round(d["ms_per_step"], 3),
      "e2e", round(d["e2e"]["value"]),
      {k: (round(v["ms_per_launch"], 4), v["launches"]) for k, v in d["kernels"].items() if v["launches"]})
PY
  IFS=';'
done
