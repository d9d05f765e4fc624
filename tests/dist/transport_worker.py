"""2-rank gloo check of sharded.alltoall_packets with the engine's packet
layout (int32 lane counts padded to 32 B, then 32 B records), built from a
real shard plan: every rank must receive exactly its import lanes' packets."""

import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

from paper_2405_12520_b200 import EngineConfig, generate_grid  # noqa: E402
from paper_2405_12520_b200 import shard  # noqa: E402
from paper_2405_12520_b200.flat import flatten_network  # noqa: E402
from paper_2405_12520_b200.sharded import alltoall_packets  # noqa: E402


def packet(lanes, rank):
    counts = (np.asarray(lanes) % 3).astype(np.int32)  # deterministic per lane
    head = counts.tobytes()
    head += b"\0" * ((-len(head)) % 32)
    recs = b"".join(np.array([lane, rank, k, 7], dtype=np.int64).tobytes()
                    for lane, c in zip(lanes, counts) for k in range(c))
    return head + recs


def main():
    dist.init_process_group("gloo")
    rank, ws = dist.get_rank(), dist.get_world_size()
    net = generate_grid(5, 5, lanes_per_direction=2)
    flat = flatten_network(net)
    jp = np.array([net.junctions[j].position for j in flat.junction_ids], dtype=np.float64)
    plan = shard.plan_all(flat, jp, ws, EngineConfig())[rank]
    pk = [packet(plan.export_lanes[q], rank) if q != rank else b"" for q in range(ws)]
    out_b = np.array([len(x) for x in pk], dtype=np.int64)
    send = torch.frombuffer(bytearray(b"".join(pk) + b"\0"), dtype=torch.uint8)
    recv = torch.zeros(1 << 20, dtype=torch.uint8)
    got, in_b = alltoall_packets(send, out_b, recv, None, False)
    ok = True
    off = 0
    for q in range(ws):
        exp = packet(plan.import_lanes[q], q) if q != rank else b""
        ok &= bytes(got[off:off + in_b[q]].numpy().tobytes()) == exp
        off += in_b[q]
    t = torch.tensor([1 if ok else 0])
    dist.all_reduce(t)
    if rank == 0:
        print(f"TRANSPORT_OK {int(t.item())}", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
