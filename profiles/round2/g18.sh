mkdir -p gpurun_out
TSB_TRACE_ERRORS=1 timeout 600 python -m pytest -q -s -m gpu tests/test_gpu_golden.py -k control_surface --timeout 300 > gpurun_out/g18_cs.log 2>&1; echo cs rc $?
