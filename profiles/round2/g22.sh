mkdir -p gpurun_out
T=g22
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_shard.py --timeout 1200 --durations=5 > gpurun_out/${T}_shard.log 2>&1; echo shard rc $?
timeout 900 python tools/rank_step_bench.py 8 0,3 > gpurun_out/${T}_rank8.txt 2> gpurun_out/${T}_rank8.err; echo rank8 rc $?
timeout 900 python tools/rank_step_bench.py 4 1 > gpurun_out/${T}_rank4.txt 2> gpurun_out/${T}_rank4.err; echo rank4 rc $?
timeout 900 python tools/rank_step_bench.py 2 0 > gpurun_out/${T}_rank2.txt 2> gpurun_out/${T}_rank2.err; echo rank2 rc $?
