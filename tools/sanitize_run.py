"""Scenario driver for compute-sanitizer runs (profiles/*sanitize*.log):
C1 (4x4 grid, 1k trips) and the dense revert-chain grid of
tests/test_gpu_parity.py through every resolver path, plus the device
queries.  Usage: python tools/sanitize_run.py [steps] [extra debug bits]"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2405_12520_b200 import EngineConfig, World, _native, generate_grid, random_trips  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    extra = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # debug bits added to every case (8: no conditional nodes)
    cases = [("C1", generate_grid(4, 4), 1000, 42, (0.0, 3600.0), 0)]
    dense = generate_grid(6, 6, block_length=60.0)
    for dbg in (0, 1, 2, 4, 8, 64):
        cases.append((f"dense_short_blocks/debug{dbg}", dense, 6000, 5, (0.0, 200.0), dbg))
    for name, net, n, seed, window, dbg in cases:
        trips = random_trips(net, n, seed=seed, window=window)
        w = World(net, trips, EngineConfig(), seed=seed)
        if dbg | extra:
            _native.check(_native.lib().tsb_set_debug(w._h, dbg | extra))
        w.run(steps)
        w.records_arrays()
        w.get_vehicle(trips[0].id)
        w.min_front_gap()
        w.road_windows(w.time)
        print(f"{name}: {steps} steps, driving {w.driving_count()}, reverts {w._report.reverts_total}", flush=True)
        w.close()


if __name__ == "__main__":
    main()
