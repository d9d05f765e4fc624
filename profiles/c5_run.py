"""C5 scale on ONE GPU: generate_grid(200,200,block_length=400,lanes_per_direction=3)
(built by the native grid builder, gridgen.grid_flat)
with N pre-placed routable vehicles (22 slots/lane at 17.6 m,
first 10,000,000), EngineConfig defaults; bulk injection step, warm-up, then
K graph-replayed steps timed with CUDA events.  Prints one JSON line."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2405_12520_b200 import EngineConfig, Router, World, _native, preplaced_trips  # noqa: E402
from paper_2405_12520_b200.flat import flatten_trips  # noqa: E402
from paper_2405_12520_b200.gridgen import grid_flat  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
t0 = time.time()
flat, _ = grid_flat(200, 200, block_length=400.0, lanes_per_direction=3)  # native builder (sha-pinned)
t_net = time.time()
router = Router(None, flat=flat)
trips = preplaced_trips(flat, router, n, 17.6)
router.close()
ft = flatten_trips(flat, trips)
t1 = time.time()
w = World.from_flat(flat, ft, EngineConfig(), seed=42, pow_mode=0)
t2 = time.time()
w.step()
drv = w.driving_count()
w.run(10)
L = _native.lib()
ms = C.c_double()
u0 = w.vehicle_updates
_native.check(L.tsb_time_steps(w._h, steps, C.byref(ms)))
_native.check(L.tsb_report_get(w._h, C.byref(w._report)))
u = w.vehicle_updates - u0
print(json.dumps({"workload": f"C5 scale: generate_grid(200,200,400 m,3 lanes), {len(trips)} pre-placed routable trips "
                  f"(17.6 m slots)", "lanes": flat.n_lanes, "driving_after_injection": drv, "steps": steps,
                  "ms_per_step": ms.value / steps, "vehicle_updates_per_s": u / (ms.value / 1e3),
                  "build_inputs_s": round(t1 - t0, 1), "build_network_s": round(t_net - t0, 1), "engine_create_s": round(t2 - t1, 1)}), flush=True)
