# full GPU suite (durations) + default bench, after the tile-sum fusion
mkdir -p gpurun_out
T=g4
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
timeout 3300 python -m pytest -q -m gpu tests --timeout 1200 --durations=40 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
