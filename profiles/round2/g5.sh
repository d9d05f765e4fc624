# sharded max-pressure tests, compute-sanitizer runs, step time vs size (cost model)
mkdir -p gpurun_out
T=g5
timeout 1500 python -m pytest -q -m gpu tests/test_gpu_shard.py -k "max_pressure or equals_single" --timeout 900 --durations=10 > gpurun_out/${T}_shard.log 2>&1; echo shard rc $?
timeout 900 compute-sanitizer --tool memcheck --leak-check full --error-exitcode 9 python tools/sanitize_run.py 60 > gpurun_out/${T}_memcheck.log 2>&1; echo memcheck rc $?
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --error-exitcode 9 python tools/sanitize_run.py 25 > gpurun_out/${T}_racecheck.log 2>&1; echo racecheck rc $?
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_run.py 25 > gpurun_out/${T}_synccheck.log 2>&1; echo synccheck rc $?
for n in 125000 250000 500000 1000000; do
  timeout 600 python bench.py --vehicles $n --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_size_$n.json 2> gpurun_out/${T}_size_$n.err; echo size $n rc $?
done
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_place|k_lanefix|k_resolve_fast|k_regroup|k_scan" -s 10 -c 5 -o gpurun_out/${T}_chain \
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_chain.log 2>&1; echo ncu chain rc $?
