mkdir -p gpurun_out
VARIANTS="base10 spat1 spat2 spat1_296" sh profiles/round2/abv.sh > gpurun_out/g33_ab.txt 2>&1; echo ab rc $?
python - >> gpurun_out/g33_ab.txt <<'PY'
import json
for v in ("base10", "spat1", "spat2", "spat1_296"):
    x = json.load(open(f"gpurun_out/abv_{v}_1.json"))
    print(v, {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()}, round(x["e2e"]["value"] / 1e9, 3))
PY
