mkdir -p gpurun_out
VARIANTS="base11 sidefused" sh profiles/round2/abv.sh > gpurun_out/g34_ab.txt 2>&1; echo ab rc $?
VARIANTS="sidefused base11" sh profiles/round2/abv.sh > gpurun_out/g34_ab2.txt 2>&1; echo ab rc $?
python - >> gpurun_out/g34_ab.txt <<'PY'
import json
for v in ("base11", "sidefused"):
    x = json.load(open(f"gpurun_out/abv_{v}_1.json"))
    print(v, {p: round(t, 1) for p, t in x["phases_us_in_graph"].items()}, round(x["e2e"]["value"] / 1e9, 3))
PY
TSB200_LIB=$PWD/build_variants/lib_sidefused.so timeout 1200 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_random.py "tests/test_gpu_configs.py::test_m1_into_the_revert_regime" --timeout 900 > gpurun_out/g34_pytest.log 2>&1; echo pytest rc $?
