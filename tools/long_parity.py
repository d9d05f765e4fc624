"""Long-run parity evidence at the bench scales (one-off, not a test):
M1 (1M vehicles) for N steps and C5 scale (200x200x3, 7M vehicles) for a
few, GPU engine vs the CPU oracle in the reference's arithmetic (glibc pow),
every StepReport counter each step, the whole lane-sorted state every K
steps.  Prints one line per checkpoint and a final JSON summary.
Usage: python tools/long_parity.py [m1_steps] [c5_steps]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle.bind import OracleWorld  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, Router, World, preplaced_trips  # noqa: E402
from paper_2405_12520_b200.flat import flatten_trips  # noqa: E402
from paper_2405_12520_b200.gridgen import grid_flat  # noqa: E402
from tests.parity import compare_reports, compare_state  # noqa: E402


def run(tag, rows, n, spacing, steps, every):
    flat, _ = grid_flat(rows, rows, 400.0, 3)
    router = Router(None, flat=flat)
    trips = preplaced_trips(flat, router, n, spacing)
    router.close()
    ft = flatten_trips(flat, trips)
    g = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=1)
    o = OracleWorld(None, trips, EngineConfig(), seed=42, pow_mode=1, flat=flat)
    o.set_threads(os.cpu_count() or 1)
    reverts, t0 = 0, time.time()
    for k in range(1, steps + 1):
        g.step()
        o.step(1)
        reverts += o.report().reverts_last
        compare_reports(g, o, k)
        if k % every == 0 or k == steps:
            compare_state(g, o, k)
            print(f"{tag} step {k}: identical (driving {g.driving_count()}, reverts so far {reverts}, "
                  f"{time.time() - t0:.0f} s)", flush=True)
    assert g.finished == o.finished_list()
    assert np.array_equal(g._state()["status"], o.status()[0])
    out = {"workload": tag, "vehicles": len(trips), "steps": steps, "reverts": int(reverts),
           "result": "bit-identical every step (reports) and every %d steps (state)" % every}
    g.close()
    o.close()
    return out


def main():
    m1 = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    c5 = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    res = [run("M1", 100, 1_000_000, 29.0, m1, 25)]
    if c5:
        res.append(run("C5", 200, 10_000_000, 17.6, c5, 1))
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
