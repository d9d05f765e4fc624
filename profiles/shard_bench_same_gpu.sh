# 2 ranks sharing one GPU (functional check of bench.py's N>1 path; time-sliced, not a scaling number)
mkdir -p gpurun_out
for X in p2p nccl; do
TSB_BENCH_GLOO=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr 127.0.0.1 --master-port 29655 bench.py --gpus 2 --steps 20 --warmup 3 --exchange $X > gpurun_out/shard2_$X.json 2> gpurun_out/shard2_$X.err; echo $X rc $?
done
