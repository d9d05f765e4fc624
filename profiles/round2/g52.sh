mkdir -p gpurun_out
VARIANTS="base lxr6 lxr5" sh profiles/round2/abv.sh > gpurun_out/g52_ab.txt 2>&1; echo ab rc $?
cat gpurun_out/g52_ab.txt
for v in base lxr6 lxr5; do python - $v <<'PY'
import json,sys
v=sys.argv[1]
for k in (1,2):
    x=json.loads(open(f"gpurun_out/abv_{v}_{k}.json").read().strip().splitlines()[-1])
    print(v, k, {a: round(b,1) for a,b in x["phases_us_in_graph"].items()})
PY
done
TSB200_LIB=$PWD/build_variants/lib_lxr6.so timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py > gpurun_out/g52_pytest.txt 2>&1; echo pytest rc $?
tail -3 gpurun_out/g52_pytest.txt
