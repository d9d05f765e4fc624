# usage: gpu_iter.sh TAG  -- parity tests, bench, ncu full on k_update
T=$1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo pytest rc $?
timeout 600 python bench.py --steps 100 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_bench.log 2>&1; echo bench rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${2:-k_update}" -s ${3:-4} -c 1 -o gpurun_out/${T}_full python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1; echo full rc $?
