mkdir -p gpurun_out
T=g7
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py 25 8 > gpurun_out/${T}_synccheck_gated.log 2>&1; echo synccheck gated rc $?
timeout 1200 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 25 8 > gpurun_out/${T}_racecheck_gated.log 2>&1; echo racecheck gated rc $?
timeout 900 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_run.py 60 8 > gpurun_out/${T}_memcheck_gated.log 2>&1; echo memcheck gated rc $?
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_run.py 15 > gpurun_out/${T}_initcheck.log 2>&1; echo initcheck rc $?
