# A/B of libtsb200.so variants (build_variants/lib_*.so): VARIANTS="a b c" sh profiles/abv.sh
mkdir -p gpurun_out
for rep in 1 2; do for v in $VARIANTS; do
  TSB200_LIB=$PWD/build_variants/lib_$v.so timeout 300 python bench.py --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/abv_${v}_$rep.json 2> gpurun_out/abv_${v}_$rep.err
done; done
for v in $VARIANTS; do python - "$v" <<'PY'
import json, sys
v = sys.argv[1]
out = []
for k in (1, 2):
    try:
        x = json.loads(open(f"gpurun_out/abv_{v}_{k}.json").read().strip().splitlines()[-1])
        out.append((round(x["ms_per_step"], 4), round(x["phases_us_in_graph"].get("update", 0), 1),
                    round(x["config"]["pow"].get("value_pow_glibc", 0) / 1e9, 3)))
    except Exception as exc:
        out.append(repr(exc)[:80])
print(v, out, flush=True)
PY
done
