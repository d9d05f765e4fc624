mkdir -p gpurun_out
T=g6
timeout 1800 python -m pytest -q -m gpu tests/test_gpu_shard.py tests/test_gpu_queries.py tests/test_gpu_parity.py tests/test_gpu_golden.py --timeout 900 --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
VARIANTS="flags placelist" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py 25 > gpurun_out/${T}_synccheck.log 2>&1; echo synccheck rc $?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 25 > gpurun_out/${T}_racecheck.log 2>&1; echo racecheck rc $?
