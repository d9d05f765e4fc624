mkdir -p gpurun_out
T=g10
timeout 1500 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py 200 > gpurun_out/${T}_synccheck_graph.log 2>&1; echo synccheck graph rc $?
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 200 > gpurun_out/${T}_racecheck_graph.log 2>&1; echo racecheck graph rc $?
VARIANTS="cur cur_lx5 cur_stream" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shard.py --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
