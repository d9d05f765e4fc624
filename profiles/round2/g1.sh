mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/g1_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo smoke rc $?
timeout 1800 python -m pytest tests -q -m gpu -x --timeout 900 > gpurun_out/g1_pytest.log 2>&1; echo pytest rc $?
timeout 900 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo bench rc $?
