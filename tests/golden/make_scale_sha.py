"""sha256 of the reference's flattened M1/C5 grids (run in the dev container,
where /root/reference exists): trafficsim.network.generate_grid(100, 100,
block_length=400, lanes_per_direction=3) and (200, 200, ...), flattened with
paper_2405_12520_b200.flat.flatten_network (which duck-types the reference's
types).  Pins the native grid builder (csrc/gridgen.cpp, tests/test_gridgen.py)
at the bench scales without committing ~100 MB of arrays."""

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, "/root/reference/pkg/src")

from trafficsim.network import generate_grid  # noqa: E402  (the reference)

from paper_2405_12520_b200.flat import flatten_network  # noqa: E402
from tests.goldens import NET_FIELDS  # noqa: E402


def flat_sha(f) -> str:
    h = hashlib.sha256()
    h.update(str(f.n_lanes).encode())
    h.update("\n".join(f.road_ids).encode())
    h.update("\n".join(f.junction_ids).encode())
    for k in NET_FIELDS:
        a = getattr(f, k)
        h.update(k.encode())
        h.update(a.dtype.str.encode())
        h.update(a.tobytes())
    return h.hexdigest()


def main():
    out = {}
    for rows, cols in ((100, 100), (200, 200)):
        t0 = time.time()
        net = generate_grid(rows, cols, block_length=400.0, lanes_per_direction=3)
        for ctl in ("fixed", "max_pressure"):
            f = flatten_network(net, ctl)
            out[f"grid{rows}x{cols}_400_3_{ctl}"] = {"sha256": flat_sha(f), "n_lanes": f.n_lanes}
        print(rows, cols, f"{time.time() - t0:.1f} s", flush=True)
        del net
    with open(os.path.join(HERE, "scale_sha.json"), "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
