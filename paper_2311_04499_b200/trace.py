"""Real-timeline profiler of the overlapped schedule.

``record_step`` turns on CUDA-event recording in a ``CovapSync``'s state,
runs one overlapped step through a caller-supplied function and returns the
per-bucket timeline (K1 start/end on the producing stream, collective
start/end and K2 end on the side stream).  ``chrome_trace`` writes it in the
reference's Chrome-trace format (report.cpp:210-230: complete events, tid 0
compute / 1 comm, µs), and ``model_check`` feeds the measured per-bucket
times into the reference's overlap_schedule (perf.cpp:63-103) so predicted
and measured step time / exposure can be compared.
"""
from __future__ import annotations

import ctypes
import json
from typing import Callable, Dict, List, Optional, Sequence

from . import _lib as L
from .covap import CovapSync, overlap_schedule


def record_step(sync: CovapSync, run_step: Callable[[], None]) -> List[Dict[str, float]]:
    """Run one step with event recording on; return one row per bucket."""
    L.lib().covap_state_set_timeline(sync.state.handle, 1)
    try:
        run_step()
        n = len(sync.plan.buckets)
        rows = (ctypes.c_double * (5 * n))()
        L.lib().covap_state_timeline(sync.state.handle, rows, n)
    finally:
        L.lib().covap_state_set_timeline(sync.state.handle, 0)
    keys = ("k1_start", "k1_end", "comm_start", "comm_end", "k2_end")
    return [{k: rows[5 * b + i] for i, k in enumerate(keys)} for b in range(n)]


def chrome_trace(path: str, timeline: Sequence[Dict[str, float]], rank: int = 0,
                 compute_blocks: Optional[Sequence[tuple]] = None, label: str = "covap"):
    """Write the timeline as a Chrome trace (chrome://tracing, Perfetto)."""
    ev = []
    for b, row in enumerate(timeline):
        ev.append({"name": f"{label} K1 b{b}", "ph": "X", "ts": row["k1_start"] * 1e3,
                   "dur": (row["k1_end"] - row["k1_start"]) * 1e3, "pid": rank, "tid": 0,
                   "args": {"bucket": b}})
        if row["comm_start"] >= 0:
            ev.append({"name": f"{label} allreduce b{b}", "ph": "X", "ts": row["comm_start"] * 1e3,
                       "dur": (row["comm_end"] - row["comm_start"]) * 1e3, "pid": rank, "tid": 1,
                       "args": {"bucket": b}})
            ev.append({"name": f"{label} K2 b{b}", "ph": "X", "ts": row["comm_end"] * 1e3,
                       "dur": (row["k2_end"] - row["comm_end"]) * 1e3, "pid": rank, "tid": 1,
                       "args": {"bucket": b}})
    for name, start_ms, end_ms in compute_blocks or ():
        ev.append({"name": name, "ph": "X", "ts": start_ms * 1e3, "dur": (end_ms - start_ms) * 1e3,
                   "pid": rank, "tid": 0})
    with open(path, "w") as f:
        json.dump({"traceEvents": ev, "displayTimeUnit": "ms"}, f, indent=1)


def model_check(timeline: Sequence[Dict[str, float]], comp_ms: Sequence[float],
                measured_step_ms: float) -> Dict[str, float]:
    """Predicted (overlap_schedule over the measured per-bucket K1 and
    collective+K2 times) vs measured step time and exposure."""
    compress = [r["k1_end"] - r["k1_start"] for r in timeline]
    comm = [max(0.0, r["k2_end"] - r["comm_start"]) if r["comm_start"] >= 0 else 0.0
            for r in timeline]
    sent = [r["comm_start"] >= 0 for r in timeline]
    sc = overlap_schedule(0.0, comp_ms, compress, comm, sent)
    return {"predicted_step_ms": sc.total_ms, "predicted_exposed_ms": sc.unoverlapped_comm_ms,
            "measured_step_ms": measured_step_ms,
            "model_error": (measured_step_ms - sc.total_ms) / sc.total_ms if sc.total_ms else 0.0}
