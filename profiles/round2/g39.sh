mkdir -p gpurun_out
for rep in 1 2; do for d in 0 16; do
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline --debug $d > gpurun_out/g39_d${d}_$rep.json 2>/dev/null
done; done
python - <<'PY'
import json
for d in (0, 16):
    for rep in (1, 2):
        x = json.load(open(f"gpurun_out/g39_d{d}_{rep}.json"))
        print("debug", d, round(x["ms_per_step"], 4), {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()})
PY
