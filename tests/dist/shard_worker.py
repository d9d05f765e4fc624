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
    "grid6x2mp": lambda: (generate_grid(6, 6, lanes_per_direction=2), 2500, 3, (0.0, 300.0)),
    "grid8x3mp": lambda: (generate_grid(8, 8, lanes_per_direction=3), 4000, 9, (0.0, 400.0)),
    "dense": lambda: (generate_grid(6, 6, block_length=80.0, lanes_per_direction=2), 5000, 5, (0.0, 200.0)),
    "grid8x3": lambda: (generate_grid(8, 8, lanes_per_direction=3), 4000, 9, (0.0, 400.0)),
}


def scenario(name):
    """(net, trips, seed) of a named scenario; "m1" is bench.py's workload
    (100x100x3 grid, 1M pre-placed routable vehicles)."""
    if name == "m1":
        from paper_2405_12520_b200 import Router, preplaced_trips

        net = generate_grid(100, 100, block_length=400.0, lanes_per_direction=3)
        router = Router(net)
        trips = preplaced_trips(net, router, 1_000_000, 29.0)
        router.close()
        return net, trips, 42
    net, n, seed, window = SCEN[name]()
    return net, random_trips(net, n, seed=seed, window=window), seed


def agree_bad(bad: int) -> int:
    """Mismatch count summed over ranks: every rank stops at the same step
    (a rank-local break would leave its peers waiting in a collective)."""
    import torch

    t = torch.tensor([bad])
    dist.all_reduce(t)
    return int(t.item())


def stall_test():
    """Rank 1 stops stepping; rank 0's bounded device-side wait for rank 1's
    exchange flag must end the step with TSB_ECUDA (EngineError), not hang."""
    from paper_2405_12520_b200.errors import EngineError

    rank, ws = dist.get_rank(), dist.get_world_size()
    net, trips, seed = scenario("grid6x2")
    sw = ShardedWorld.from_network(net, trips, EngineConfig(), seed=seed, rank=rank, nranks=ws, device=0,
                                   host_staging=True, p2p=True)
    assert sw.p2p, sw.p2p_error
    sw.set_p2p_timeout(0.5)
    sw.step_local(5)
    dist.barrier()
    msg = "no error"
    if rank == 0:
        try:
            sw.step_local(3)  # rank 1 is not stepping
        except EngineError as exc:
            msg = str(exc)
    dist.barrier()
    sw.close()
    if rank == 0:
        ok = "did not come within" in msg
        print(f"STALL_RESULT ok={int(ok)} msg={msg!r}", flush=True)


def check_queries(sw, ref, rank, k) -> int:
    """The merged query surface of the sharded engine (collective) against the
    single engine: id-sorted records with headings, arrivals in reference
    order, road windows, and get_vehicle for a sample of ids."""
    bad = 0
    a, b = sw.records_arrays(), ref.records_arrays()
    for key in ("vix", "lane", "road_pos", "s", "v", "angle_deg"):
        if not np.array_equal(a[key], b[key]):
            print(f"rank {rank} step {k}: records field {key} differs", flush=True)
            bad += 1
            break
    if sw.finished != ref.finished:
        print(f"rank {rank} step {k}: finished lists differ ({len(sw.finished)} vs {len(ref.finished)})", flush=True)
        bad += 1
    if sw.road_windows(ref.time) != ref.road_windows(ref.time):
        print(f"rank {rank} step {k}: road windows differ", flush=True)
        bad += 1
    rng = np.random.default_rng(k)
    ids = ref._ft.ids
    for i in rng.choice(len(ids), min(25, len(ids)), replace=False).tolist():
        got = sw.get_vehicle(ids[i])  # collective: every rank makes every call
        if got != ref.get_vehicle(ids[i]):
            print(f"rank {rank} step {k}: get_vehicle({ids[i]}) differs: {got} vs {ref.get_vehicle(ids[i])}",
                  flush=True)
            bad += 1
    return bad


def main():
    name, steps = sys.argv[1], int(sys.argv[2])
    p2p = len(sys.argv) > 3 and sys.argv[3] == "p2p"
    dist.init_process_group("gloo")
    if name == "stall":
        stall_test()
        dist.destroy_process_group()
        return
    rank, ws = dist.get_rank(), dist.get_world_size()
    net, trips, seed = scenario(name)
    cfg = EngineConfig(controller="max_pressure") if name.endswith("mp") else EngineConfig()
    sw = ShardedWorld.from_network(net, trips, cfg, seed=seed, rank=rank, nranks=ws, device=0, host_staging=True,
                                   p2p=p2p, local_lanes=os.environ.get("TSB_SHARD_GLOBAL_LANES") != "1")
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
        if k % 50 == 0 or k == steps:
            bad += check_queries(sw, ref, rank, k)
        if agree_bad(bad):
            break
    ex = sw.exchange_bytes()
    used_p2p = sw.p2p
    sw.close()
    ref.close()
    total_bad = agree_bad(bad)
    if rank == 0:
        print(f"SHARD_RESULT {name} ranks={ws} steps={steps} p2p={int(p2p)} p2p_used={int(used_p2p)} "
              f"mismatches={total_bad} "
              f"bytes_rank0={ex}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
