"""Per-phase timeline of graph-replayed steps on the M1 workload (bench.py's).

Turns the step timeline on (tsb_set_timeline: every step kernel's block 0
stamps %globaltimer when it passes its dependency wait), runs 20 + 40 steps
and prints, for the last 40, the median offset (us) of each phase's start
from the step's begin kernel, the median in-graph phase durations and the
median step period.  Measurement tool, not a test.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, World, _native  # noqa: E402

PH = ["begin", "update", "scan", "place", "lanefix", "resolve_fast", "regroup", "end", "speeds", "signals",
      "inject_due", "speeds_end", "resolve_fast_end", "inject_due_end"]
n = int(os.environ.get("TSB_VEHICLES", "1000000"))
net, flat, trips, ft, _ = bench.build_workload(n, 29.0)
w = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=int(os.environ.get("TSB_POW", "0")))
L = _native.lib()
if os.environ.get("TSB_DEBUG"):
    _native.check(L.tsb_set_debug(w._h, int(os.environ["TSB_DEBUG"])))
_native.check(L.tsb_set_timeline(w._h, 1))
w.step()
w.run(20)
w.run(40)
rows = bench.timeline_rows(L, w._h, 40)
off = {}
for k, name in enumerate(PH):
    vals = [(r[k] - r[0]) / 1000.0 for r in rows if r[k] > 0]
    if vals:
        off[name] = round(float(np.median(vals)), 2)
dur, period = bench.phase_durations(rows)
pct = {k: [round(float(np.percentile(v, q)), 1) for q in (10, 50, 90)] for k, v in dur.items()}
starts = {name: [round((r[k] - r[0]) / 1000.0, 1) if r[k] > 0 else None for r in rows[:8]] for k, name in enumerate(PH)}
out = {"phase_start_us_median": off, "phase_us_p10_p50_p90": pct, "first_8_steps_phase_starts_us": starts,
       "phase_us_median": {k: round(float(np.median(v)), 2) for k, v in dur.items()},
       "step_period_us_median": round(float(np.median(period)), 2), "steps": len(rows)}
print(json.dumps(out))
