mkdir -p gpurun_out
VARIANTS="base9 sp148 sp74 sp296" sh profiles/round2/abv.sh > gpurun_out/g32_ab.txt 2>&1; echo ab rc $?
python - >> gpurun_out/g32_ab.txt <<'PY'
import json
for v in ("base9", "sp148", "sp74", "sp296"):
    x = json.load(open(f"gpurun_out/abv_{v}_1.json"))
    print(v, {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()})
PY
