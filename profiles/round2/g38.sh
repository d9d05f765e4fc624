mkdir -p gpurun_out
timeout 3300 python tools/long_parity.py 1000 10 > gpurun_out/g38_long_parity.log 2>&1; echo long rc $?
timeout 900 python -m pytest -q -m gpu "tests/test_gpu_configs.py::test_m1_into_the_revert_regime" --timeout 900 -s > gpurun_out/g38_m1.log 2>&1; echo m1 rc $?
