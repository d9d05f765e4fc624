# round 2 call 2: parity of the side-compacted k_update, A/B of update variants, ncu of k_update
mkdir -p gpurun_out
T=g2
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err; echo bench rc $?
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_queries.py \
  tests/test_gpu_shard.py -x --timeout 900 --durations=25 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
VARIANTS="orig compact compact_m5 compact_128x8" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_update" -s 20 -c 1 -o gpurun_out/${T}_upd \
  python bench.py --steps 30 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_ncu_upd.log 2>&1; echo ncu rc $?
