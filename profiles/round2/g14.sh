mkdir -p gpurun_out
T=g14
VARIANTS="nofused fused" sh profiles/round2/abv.sh > gpurun_out/${T}_ab.txt 2>&1; echo ab rc $?
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_shard.py "tests/test_gpu_configs.py::test_m1_into_the_revert_regime" "tests/test_gpu_configs.py::test_c3_grid50_200k" --timeout 900 > gpurun_out/${T}_pytest.log 2>&1; echo pytest rc $?
TSB_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 2 --weak --vehicles 200000 --steps 5 --warmup 3 > gpurun_out/${T}_weak2.log 2>&1; echo weak rc $?
