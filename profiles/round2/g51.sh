mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g51_smoke.log 2>&1; echo smoke rc $?
timeout 3000 python -m pytest -q -m gpu tests --timeout 1200 --durations=10 > gpurun_out/g51_pytest.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/g51_pytest.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/final2_smi.txt
timeout 1200 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; echo bench rc $?
timeout 1200 python bench.py --impl reference > gpurun_out/final2_bench_reference.json 2> gpurun_out/final2_bench_reference.err; echo ref rc $?
timeout 600 python profiles/timeline.py > gpurun_out/final2_timeline.json 2> gpurun_out/final2_timeline.err; echo tl rc $?
