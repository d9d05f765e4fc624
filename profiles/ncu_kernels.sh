# usage: ncu_kernels.sh TAG -- one --set full capture of each steady-state
# step kernel after the update (scan, place, lanefix, fast resolve, regroup)
T=$1
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_place|k_lanefix|k_resolve_fast|k_regroup|k_scan" -s 20 -c 6 -o gpurun_out/${T}_kern python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_kern.log 2>&1; echo kern rc $?
