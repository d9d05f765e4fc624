"""Worker for tests/test_gpu_shard.py: N ranks (torchrun), each a shard of the
engine, compared step by step with a single-GPU engine on the same inputs.

Run: python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1
     --master-port P tests/dist/shard_worker.py SCENARIO STEPS
All ranks may share one GPU (gloo exchange with host staging; with a third
argument "p2p" the device-driven exchange over CUDA IPC-mapped peer memory).
"""

from __future__ import annotations

import os
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2405_12520_b200 import EngineConfig, World, generate_grid, random_trips  # noqa: E402
from paper_2405_12520_b200.sharded import ShardedWorld  # noqa: E402

SCEN = {
    "grid6x2": lambda: (generate_grid(6, 6, lanes_per_direction=2), 1500, 3, (0.0, 300.0)),
    "dense": lambda: (generate_grid(6, 6, block_length=80.0, lanes_per_direction=2), 5000, 5, (0.0, 200.0)),
    "grid8x3": lambda: (generate_grid(8, 8, lanes_per_direction=3), 4000, 9, (0.0, 400.0)),
}


def main():
    name, steps = sys.argv[1], int(sys.argv[2])
    p2p = len(sys.argv) > 3 and sys.argv[3] == "p2p"
    dist.init_process_group("gloo")
    rank, ws = dist.get_rank(), dist.get_world_size()
    net, n, seed, window = SCEN[name]()
    trips = random_trips(net, n, seed=seed, window=window)
    cfg = EngineConfig()
    sw = ShardedWorld.from_network(net, trips, cfg, seed=seed, rank=rank, nranks=ws, device=0, host_staging=True,
                                   p2p=p2p)
    ref = World(net, trips, cfg, seed=seed)
    own_zone = sw.plan.zone
    bad = 0
    for k in range(1, steps + 1):
        sw.step_local(1)
        ref.step()
        rep = sw.report()
        rr = ref._report
        for key in ("driving", "waiting", "finished", "dropped", "injected_now", "finished_now", "vehicle_updates"):
            if rep[key] != getattr(rr, key):
                print(f"rank {rank} step {k}: {key} {rep[key]} vs {getattr(rr, key)}", flush=True)
                bad += 1
        if k % 10 == 0 or k == steps:
            mine = sw.own_state()
            st = ref._state()
            sel = (own_zone[st["lane"]] & 1) > 0
            for key, rk in (("vix", "vix"), ("lane", "lane"), ("road_pos", "rp"), ("s", "s"), ("v", "v")):
                if not np.array_equal(mine[key], st[rk][sel]):
                    print(f"rank {rank} step {k}: own-lane field {key} differs", flush=True)
                    bad += 1
                    break
        if bad:
            break
    ex = sw.exchanged_bytes
    used_p2p = sw.p2p
    sw.close()
    ref.close()
    flag = np.array([bad])
    import torch
    t = torch.tensor(flag)
    dist.all_reduce(t)
    if rank == 0:
        print(f"SHARD_RESULT {name} ranks={ws} steps={steps} p2p={int(p2p)} p2p_used={int(used_p2p)} "
              f"mismatches={int(t.item())} "
              f"bytes_rank0={ex}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
