T=r2a
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${T}_smi.txt
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
TSB200_LIB=$PWD/build_variants/lib_tl.so timeout 600 python profiles/timeline.py > gpurun_out/${T}_timeline.json 2> gpurun_out/${T}_timeline.err; echo tl rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_update" -s 20 -c 1 -o gpurun_out/${T}_upd python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_upd.log 2>&1; echo full rc $?
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_place|k_lanefix|k_resolve_fast|k_regroup|k_scan|k_tile" -s 10 -c 6 -o gpurun_out/${T}_kern python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_kern.log 2>&1; echo kern rc $?
