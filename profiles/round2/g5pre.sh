mkdir -p gpurun_out
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29701 tools/shard_query_debug.py grid6x2 50 > gpurun_out/g5_dbg1.log 2>&1; echo dbg1 rc $?
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node=3 --master-addr 127.0.0.1 --master-port 29702 tools/shard_query_debug.py grid8x3 50 p2p > gpurun_out/g5_dbg2.log 2>&1; echo dbg2 rc $?
