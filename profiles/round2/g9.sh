mkdir -p gpurun_out
T=g9
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_queries.py --timeout 1200 --durations=8 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
VARIANTS="base rcp rcp_lx5" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 200 8 > gpurun_out/${T}_racecheck_gated.log 2>&1; echo racecheck gated rc $?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 200 > gpurun_out/${T}_racecheck_graph.log 2>&1; echo racecheck graph rc $?
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py 200 > gpurun_out/${T}_synccheck_graph.log 2>&1; echo synccheck graph rc $?
