"""Timeline export in the reference's TimelineEvent schema (simulator.hpp:19-25):
Chrome trace JSON (one process, threads "load" and "compute", microsecond
timestamps) and CSV `stream,layer,expert,start_s,end_s`.  Works
for simulated timelines (simulate/simulate_model) and for the MEASURED ones the
offloaded layer returns (MoELayer.forward(..., want_timeline=True))."""
from __future__ import annotations

import json
from typing import Iterable, Sequence, Tuple

EventT = Tuple[int, int, int, float, float]
STREAMS = {0: "load", 1: "compute"}


def shift_layer(events: Iterable[EventT], layer: int, t0: float) -> list:
    """Re-label one layer's measured events and offset them by t0 seconds."""
    return [(st, layer, e, a + t0, b + t0) for st, _l, e, a, b in events]


def to_chrome_trace(events: Sequence[EventT], name: str = "infmoe") -> dict:
    tr = [{"ph": "M", "pid": 0, "name": "process_name", "args": {"name": name}}]
    for tid, label in STREAMS.items():
        tr.append({"ph": "M", "pid": 0, "tid": tid, "name": "thread_name",
                   "args": {"name": label}})
    for st, l, e, a, b in events:
        tr.append({"ph": "X", "pid": 0, "tid": int(st), "name": f"L{l}/E{e}",
                   "ts": a * 1e6, "dur": (b - a) * 1e6,
                   "args": {"layer": int(l), "expert": int(e)}})
    return {"traceEvents": tr, "displayTimeUnit": "ms"}


def to_csv(events: Sequence[EventT]) -> str:
    rows = ["stream,layer,expert,start_s,end_s"]
    for st, l, e, a, b in events:
        rows.append(f"{STREAMS[int(st)]},{int(l)},{int(e)},{a:.9f},{b:.9f}")
    return "\n".join(rows) + "\n"


def write(events: Sequence[EventT], path_prefix: str, name: str = "infmoe") -> None:
    with open(path_prefix + ".trace.json", "w") as fh:
        json.dump(to_chrome_trace(events, name), fh)
    with open(path_prefix + ".csv", "w") as fh:
        fh.write(to_csv(events))
