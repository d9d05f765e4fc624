mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g49_smoke.log 2>&1; echo smoke rc $?
timeout 3000 python -m pytest -q -m gpu tests --timeout 1200 --durations=10 > gpurun_out/g49_pytest.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/g49_pytest.log
bash profiles/round2/final.sh
timeout 600 python profiles/timeline.py > gpurun_out/final_timeline.json 2> gpurun_out/final_timeline.err; echo tl rc $?
