mkdir -p gpurun_out
VARIANTS="base rg74 rg296" sh profiles/round2/abv.sh > gpurun_out/g62_ab.txt 2>&1; echo ab rc $?
cat gpurun_out/g62_ab.txt
for v in base rg74 rg296; do python - $v <<'PY'
import json,sys
v=sys.argv[1]
for k in (1,2):
    x=json.loads(open(f"gpurun_out/abv_{v}_{k}.json").read().strip().splitlines()[-1])
    print(v, k, round(x["step_period_us_in_graph"],1), {a: round(b,1) for a,b in x["phases_us_in_graph"].items()})
PY
done
