mkdir -p gpurun_out
VARIANTS="base sp8 sp4" sh profiles/round2/abv.sh > gpurun_out/g57_ab.txt 2>&1; echo ab rc $?
cat gpurun_out/g57_ab.txt
for v in base sp8 sp4; do python - $v <<'PY'
import json,sys
v=sys.argv[1]
for k in (1,2):
    x=json.loads(open(f"gpurun_out/abv_{v}_{k}.json").read().strip().splitlines()[-1])
    print(v, k, round(x["step_period_us_in_graph"],1), {a: round(b,1) for a,b in x["phases_us_in_graph"].items()}, 'speeds_eager', round(x["eager_kernel_ms_per_step"]["k_speeds"]*1000,1))
PY
done
TSB200_LIB=$PWD/build_variants/lib_sp8.so timeout 2400 python -m pytest -x -q -m gpu tests --timeout 1200 > gpurun_out/g57_pytest.txt 2>&1; echo pytest rc $?
tail -3 gpurun_out/g57_pytest.txt
