mkdir -p gpurun_out
VARIANTS="base13 rfpoll" sh profiles/round2/abv.sh > gpurun_out/g40_ab.txt 2>&1; echo ab rc $?
VARIANTS="rfpoll base13" sh profiles/round2/abv.sh > gpurun_out/g40_ab2.txt 2>&1; echo ab rc $?
python - >> gpurun_out/g40_ab.txt <<'PY'
import json
for v in ("base13", "rfpoll"):
    x = json.load(open(f"gpurun_out/abv_{v}_1.json"))
    print(v, {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()})
PY
