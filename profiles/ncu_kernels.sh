# usage: ncu_kernels.sh TAG [REGEX] -- one --set full capture of each
# steady-state step kernel matching REGEX (eager profile pass of bench.py)
T=$1
R=${2:-k_place|k_lanefix|k_resolve_fast|k_regroup|k_scan}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$R" -s 10 -c ${3:-6} -o gpurun_out/${T}_kern python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_kern.log 2>&1; echo kern rc $?
