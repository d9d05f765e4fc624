mkdir -p gpurun_out
T=g23
timeout 2400 python -m pytest -q -m gpu tests/test_gpu_shard.py --timeout 1200 --durations=5 > gpurun_out/${T}_shard.log 2>&1; echo shard rc $?
TSB_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/${T}_bench2_p2p.log 2>&1; echo bench2 rc $?
