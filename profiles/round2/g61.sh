mkdir -p gpurun_out
T=g61
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 python tools/sanitize_run.py 200 8 > gpurun_out/${T}_${tool}_gated.log 2>&1; echo $tool gated rc $?
done
timeout 1500 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_run.py 200 > gpurun_out/${T}_memcheck_graph.log 2>&1; echo memcheck graph rc $?
for f in gpurun_out/${T}_*.log; do echo "$f: $(tail -1 $f)"; done
