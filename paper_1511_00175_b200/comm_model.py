"""Communication-time models of the paper, calibrated to B200 measurements.

The paper (§6, PAPER.md) costs data-parallel aggregation purely by bytes moved:
  Eq. 3  parameter server:  t = |∇W|·p / BW
  Eq. 4  reduction tree:    t = |∇W|·2·log2(p) / BW
This module evaluates those closed forms and, for planning on B200, the
per-GPU byte counts of the executors this library actually runs, with a fixed
per-call latency t0 and an effective link bandwidth fitted from measurements
(`calibrate`, least squares on t = t0 + bytes/BW):
  flat / forest  2(p−1)/p·|W| per GPU per direction (the allreduce lower bound)
  single_root    ceil(log2 p)·|W| per direction at the root (Eq. 4 counts in + out
                 serially: 2·log2 p; NVLink is full duplex)
  ps             (p−1)·|W| per direction at the server (also a worker)
This is a host-side planning tool (no GPU); the CPU oracle keeps its own,
independent copy of Eq. 3/4 (oracle/comm_model.py) and tests compare the two.
"""
from __future__ import annotations

from dataclasses import dataclass


def _levels(p: int, k: int = 2) -> int:
    if p < 1 or k < 2:
        raise ValueError("need p >= 1, k >= 2")
    levels, reach = 0, 1
    while reach < p:
        reach *= k
        levels += 1
    return levels


def eq3_param_server(grad_bytes: float, p: int, bw: float) -> float:
    """Eq. 3 as printed."""
    if p < 1:
        raise ValueError("p >= 1")
    return grad_bytes * p / bw


def eq4_reduction_tree(grad_bytes: float, p: int, bw: float, k: int = 2) -> float:
    """Eq. 4; k-ary: k·ceil(log_k p) serialized receives."""
    return grad_bytes * k * _levels(p, k) / bw


def schedule_bytes(schedule: str, grad_bytes: float, p: int) -> float:
    """Bytes on the busiest GPU link, per direction, for one fused call."""
    if p <= 1:
        return 0.0
    if schedule in ("flat", "forest"):
        return 2.0 * (p - 1) / p * grad_bytes
    if schedule == "single_root":  # root: log2 p partials in, log2 p weight copies out (full duplex)
        return 1.0 * _levels(p, 2) * grad_bytes
    if schedule == "ps":  # server: p-1 gradients in, p-1 sums out (full duplex)
        return 1.0 * (p - 1) * grad_bytes
    raise ValueError(f"unknown schedule {schedule!r}")


@dataclass
class Calibration:
    bw: float   # bytes/s per direction
    t0: float   # s per call (launch + barriers)

    def predict(self, schedule: str, grad_bytes: float, p: int) -> float:
        if p <= 1:
            return 0.0
        return self.t0 + schedule_bytes(schedule, grad_bytes, p) / self.bw


def calibrate(points) -> Calibration:
    """Fit t = t0 + bytes/BW to [(schedule, grad_bytes, p, seconds), ...]."""
    xs, ys = [], []
    for sched, gb, p, t in points:
        xs.append(schedule_bytes(sched, gb, p))
        ys.append(t)
    n = len(xs)
    if n < 2:
        raise ValueError("need >= 2 points")
    mx, my = sum(xs) / n, sum(ys) / n
    sxx = sum((x - mx) ** 2 for x in xs)
    if sxx == 0:
        raise ValueError("degenerate points")
    slope = sum((x - mx) * (y - my) for x, y in zip(xs, ys)) / sxx
    t0 = my - slope * mx
    return Calibration(bw=1.0 / slope, t0=max(t0, 0.0))
