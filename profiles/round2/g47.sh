mkdir -p gpurun_out
TSB200_LIB=$PWD/build_variants/lib_lxtrace.so timeout 600 python - > gpurun_out/g47_lx.txt 2> gpurun_out/g47_lx.err <<'PY'
import bench
from paper_2405_12520_b200 import EngineConfig, World
net, flat, trips, ft, _ = bench.build_workload(1000000, 29.0)
w = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=0)
for k in range(60):
    w.step()
PY
echo rc $?; grep "^LX" gpurun_out/g47_lx.txt | tail -12
