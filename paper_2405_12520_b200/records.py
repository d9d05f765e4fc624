"""Output record types and sinks, mirroring trafficsim/io.py:49-64, 385-440.

``record_line`` reproduces the reference's canonical JSON line byte-for-byte
(sorted keys, compact separators, shortest float repr), so a
``HashingRecorder`` over this engine's stream is directly comparable with
the reference's published determinism digest.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass

from .errors import RecorderError


@dataclass(frozen=True)
class VehicleRecord:
    t: float
    id: int
    lane: int
    s: float
    v: float
    angle_deg: float


@dataclass(frozen=True)
class RoadWindow:
    road: str
    window_start: float
    window_end: float
    mean_speed: float


def canonical_json(obj) -> str:
    return json.dumps(obj, sort_keys=True, separators=(",", ":"),
                      ensure_ascii=False, allow_nan=False)


def record_line(r: VehicleRecord) -> str:
    return canonical_json({"angle_deg": r.angle_deg, "id": r.id, "lane": r.lane,
                           "s": r.s, "t": r.t, "v": r.v}) + "\n"


class JsonlRecorder:
    def __init__(self, path):
        self._fh = open(path, "w", encoding="utf-8")
        self._fh.write(canonical_json({"producer": "trafficsim", "schema_name": "vehicle-records",
                                       "schema_version": 1}) + "\n")

    def write(self, record: VehicleRecord) -> None:
        try:
            self._fh.write(record_line(record))
        except (OSError, ValueError) as exc:
            raise RecorderError(f"record write failed: {exc}") from None

    def close(self) -> None:
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False


class HashingRecorder:
    def __init__(self):
        self._h = hashlib.sha256()
        self.count = 0

    def write(self, record: VehicleRecord) -> None:
        self._h.update(record_line(record).encode("utf-8"))
        self.count += 1

    def hexdigest(self) -> str:
        return self._h.hexdigest()


class CollectingRecorder:
    def __init__(self):
        self.records: list[VehicleRecord] = []

    def write(self, record: VehicleRecord) -> None:
        self.records.append(record)
