"""B200-native MOSS per-step vehicle loop (drop-in for trafficsim's World).

The package mirrors the reference's engine interface (trafficsim/engine);
the step itself runs in libtsb200.so (csrc/, hand-written sm_100a CUDA
behind the C-ABI of include/tsb200.h).
"""

from .demand import Trip, preplaced_trips, random_trips
from .errors import (BuildError, EngineError, InputError, NoRouteError, ParseError, RecorderError,
                     SchemaError, TrafficSimError)
from .network import (CLOSED, CONNECTOR, OPEN, ROAD, BuildOptions, Junction, Lane, RawJunction,
                      RawRoad, RoadNetwork, SignalPhase, SignalProgram, build_network, generate_grid,
                      make_corridor, make_cross, make_ring)
from .params import FIXED, MAX_PRESSURE, EngineConfig, IdmParams, MobilParams
from .records import CollectingRecorder, HashingRecorder, JsonlRecorder, RoadWindow, VehicleRecord
from .routing import Router, roads_of_route
from .world import DRIVING, DROPPED, FINISHED, WAITING, SimulationOutput, StatusView, StepReport, World, run

__version__ = "0.1.0"
