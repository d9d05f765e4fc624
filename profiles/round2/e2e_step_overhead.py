"""Host cost of World.step() at M1: the step loop through World.step() (the
reference API) against the bare tsb_step call and against the previous
StepReport construction, on one World, alternating blocks.  Measurement
tool, not a test."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
from paper_2405_12520_b200 import EngineConfig, World, _native  # noqa: E402
from paper_2405_12520_b200.world import StepReport  # noqa: E402

net, flat, trips, ft, _ = bench.build_workload(1000000, 29.0)
w = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=0)
w.run(10)
L = _native.lib()


def old_step():
    _native.check(L.tsb_step(w._h, 1, C.byref(w._report)))
    r = w._report
    return StepReport(time=r.time, driving=int(r.driving), waiting=int(r.waiting), finished=int(r.finished),
                      dropped=int(r.dropped), injected_now=int(r.injected_now), finished_now=int(r.finished_now))


def bare():
    L.tsb_step(w._h, 1, None)


res = {"new": [], "old": [], "bare": []}
fns = (("new", w.step), ("old", old_step), ("bare", bare))
for k in range(600):
    name, fn = fns[k % 3]
    t0 = time.perf_counter()
    fn()
    res[name].append((time.perf_counter() - t0) * 1e6)
import numpy as np  # noqa: E402
print(json.dumps({k: {"median_us": round(float(np.median(v)), 2), "mean_us": round(float(np.mean(v)), 2)}
                  for k, v in res.items()}))
