mkdir -p gpurun_out
timeout 1800 python -m pytest -q -m gpu tests/test_gpu_random.py --timeout 600 -s > gpurun_out/g26_random.log 2>&1; echo random rc $?
bash profiles/round2/final.sh
