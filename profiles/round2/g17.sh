mkdir -p gpurun_out
T=g17
TSB_TRACE_ERRORS=1 timeout 600 python -m pytest -q -s -m gpu tests/test_gpu_golden.py -k control_surface --timeout 300 > gpurun_out/${T}_cs.log 2>&1; echo cs rc $?
TSB_TRACE_ERRORS=1 CUDA_LAUNCH_BLOCKING=1 timeout 600 python -m pytest -q -s -m gpu tests/test_gpu_golden.py -k control_surface --timeout 300 > gpurun_out/${T}_cs_blocking.log 2>&1; echo cs blocking rc $?
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
