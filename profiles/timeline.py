"""Per-phase timeline of graph-replayed steps on the M1 workload (bench.py's).

Needs a library built with -DTSB_TIMELINE (TSB200_LIB=...); prints, for the
last 40 steps, the median offset (us) of each phase's start from the step's
begin kernel and the median step period.  Measurement tool, not a test.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, World, _native  # noqa: E402

PH = ["begin", "update", "scan", "place", "lanefix", "resolve_fast", "regroup", "end", "speeds", "signals",
      "inject_due"]
net, flat, trips, ft = bench.build_workload(1_000_000, 29.0)
w = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=0)
if os.environ.get("TSB_DEBUG"):
    _native.check(_native.lib().tsb_set_debug(w._h, int(os.environ["TSB_DEBUG"])))
w.step()
w.run(20)
w.run(40)
buf = np.zeros(64 * 16, dtype=np.uint64)
_native.check(_native.lib().tsb_timeline(w._h, buf.ctypes.data))
t = buf.reshape(64, 16).astype(np.int64)
rows = [r for r in t if r[0] > 0]
rows.sort(key=lambda r: r[0])
rows = rows[-41:]
off = {}
for k, name in enumerate(PH):
    vals = [(r[k] - r[0]) / 1000.0 for r in rows[:-1] if r[k] > 0]
    if vals:
        off[name] = round(float(np.median(vals)), 2)
period = [(rows[i + 1][0] - rows[i][0]) / 1000.0 for i in range(len(rows) - 1)]
out = {"phase_start_us_median": off, "step_period_us_median": round(float(np.median(period)), 2),
       "steps": len(rows) - 1}
print(json.dumps(out))
