"""Debug helper: sharded records vs single engine (torchrun, gloo, one GPU)."""
import os
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests.dist.shard_worker import scenario  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, World  # noqa: E402
from paper_2405_12520_b200.sharded import ShardedWorld  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    name, steps = sys.argv[1], int(sys.argv[2])
    net, trips, seed = scenario(name)
    sw = ShardedWorld.from_network(net, trips, EngineConfig(), seed=seed, rank=rank, nranks=dist.get_world_size(),
                                   device=0, host_staging=True, p2p=len(sys.argv) > 3)
    ref = World(net, trips, EngineConfig(), seed=seed)
    for k in range(steps):
        sw.step_local(1)
        ref.step()
    a, b = sw.records_arrays(), ref.records_arrays()
    mine = sw.own_state()
    st = ref._state()
    sa, sb = set(a["vix"].tolist()), set(b["vix"].tolist())
    if rank == 0:
        print("sharded", len(a["vix"]), "single", len(b["vix"]), "only sharded", sorted(sa - sb)[:10],
              "only single", sorted(sb - sa)[:10], flush=True)
        dup = np.unique(a["vix"], return_counts=True)
        print("duplicates", dup[0][dup[1] > 1][:10], flush=True)
    bad = sorted((sa ^ sb))[:5]
    for x in bad:
        p = np.nonzero(st["vix"] == x)[0]
        lane_single = int(st["lane"][p[0]]) if len(p) else None
        q = np.nonzero(mine["vix"] == x)[0]
        print(f"rank {rank}: vix {x} single lane {lane_single} zone {sw.plan.zone[lane_single] if lane_single is not None else None}"
              f" own_state has it: {len(q)} lane {mine['lane'][q].tolist()}", flush=True)
    sw.close()
    ref.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
