# usage: ncu_update.sh TAG -- full ncu capture of one steady-state k_update, its
# warm-cache DRAM traffic (application replay, no cache flush), launch list
T=$1
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_update" -s 20 -c 1 -o gpurun_out/${T}_full python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1; echo full rc $?
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none --replay-mode application -k "regex:k_update" -s 20 -c 1 --csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_warm.log 2>&1; echo warm rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launch_bench.log 2>&1; echo launches rc $?
