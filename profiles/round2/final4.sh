mkdir -p gpurun_out
T=final4
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc $?
timeout 3000 python -m pytest -q -m gpu tests --timeout 1200 --durations=10 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
tail -2 gpurun_out/${T}_pytest.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/${T}_smi.txt
timeout 1200 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
timeout 1200 python bench.py --impl reference > gpurun_out/${T}_bench_reference.json 2> gpurun_out/${T}_bench_reference.err; echo ref rc $?
timeout 900 python bench.py --pow glibc --steps 50 --no-cpu-baseline > gpurun_out/${T}_bench_glibc.json 2> gpurun_out/${T}_bench_glibc.err; echo glibc rc $?
timeout 900 python bench.py --vehicles 2000000 --spacing 22 --steps 50 --no-cpu-baseline > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo c4 rc $?
timeout 600 python profiles/timeline.py > gpurun_out/${T}_timeline.json 2> gpurun_out/${T}_timeline.err; echo tl rc $?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_launches.log 2>&1; echo launches rc $?
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_place|k_lanefix|k_resolve_fast|k_regroup|k_scan" -s 10 -c 5 -o gpurun_out/${T}_chain python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_chain.log 2>&1; echo ncu chain rc $?
timeout 1500 python profiles/c5_run.py 10000000 50 > gpurun_out/${T}_c5.json 2> gpurun_out/${T}_c5.err; echo c5 rc $?
