mkdir -p gpurun_out
TSB200_LIB=$PWD/build_variants/lib_share.so timeout 900 python -m pytest -x -q -m gpu tests/test_gpu_random.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py > gpurun_out/g42_pytest.txt 2>&1; echo pytest rc $?
VARIANTS="base share" sh profiles/round2/abv.sh > gpurun_out/g42_ab.txt 2>&1; echo ab rc $?
cat gpurun_out/g42_ab.txt; tail -3 gpurun_out/g42_pytest.txt
