# usage: launches.sh TAG -- per-launch durations (ncu, serialised) of the first
# ~1500 kernel launches of a short bench run, cold (cache flush, the recipe's
# pass) and warm (--cache-control none)
T=$1
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launch_bench.log 2>&1; echo cold rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none -c 1500 --csv --log-file gpurun_out/${T}_launches_warm.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launch_bench_warm.log 2>&1; echo warm rc $?
