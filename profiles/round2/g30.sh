mkdir -p gpurun_out
VARIANTS="base8 lxrng" sh profiles/round2/abv.sh > gpurun_out/g30_ab.txt 2>&1; echo ab rc $?
VARIANTS="lxrng base8" sh profiles/round2/abv.sh > gpurun_out/g30_ab2.txt 2>&1; echo ab rc $?
python - >> gpurun_out/g30_ab.txt <<'PY'
import json
for v in ("base8", "lxrng"):
    for k in (1, 2):
        x = json.load(open(f"gpurun_out/abv_{v}_{k}.json"))
        print(v, {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()})
PY
TSB200_LIB=$PWD/build_variants/lib_lxrng.so timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py "tests/test_gpu_configs.py::test_m1_into_the_revert_regime" --timeout 900 > gpurun_out/g30_pytest.log 2>&1; echo pytest rc $?
