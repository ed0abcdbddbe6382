"""Closed-form communication-time models of the paper — TEST INFRASTRUCTURE ONLY.

Eq. 3 (§6.1):   param_server_communication_time = |∇W|·p / BW
Eq. 4 (§6.2):   reduction_tree_communication_time = |∇W|·2·log2(p) / BW

Readings (R2/R3): the formulas are implemented as printed; p=1 has no
communication; for a k-ary tree the SPEC form k·ceil(log_k p) is given
next to the counted binomial reduce+broadcast 2(k−1)·ceil(log_k p) (equal at
k=2).  ``crossover_workers`` is SPEC S:302-310.  The "counted" forms are the
byte volumes the build's schedules move per GPU (SURVEY §8 d).
"""
from __future__ import annotations


def _levels(p: int, k: int) -> int:
    if p < 1 or k < 2:
        raise ValueError("need p >= 1, k >= 2")
    L, reach = 0, 1
    while reach < p:  # integer ceil(log_k p), no floating log
        reach *= k
        L += 1
    return L


def ps_comm_time(grad_bytes: float, p: int, bw: float) -> float:
    """Eq. 3 as printed: |∇W|·p / BW."""
    if p < 1:
        raise ValueError("p >= 1")
    return grad_bytes * p / bw


def tree_comm_time(grad_bytes: float, p: int, bw: float, k: int = 2) -> float:
    """Eq. 4 for k=2; SPEC's k·ceil(log_k p) factor for k>2."""
    return grad_bytes * k * _levels(p, k) / bw


def tree_counted_factor(p: int, k: int = 2) -> int:
    """Serialized receives of a k-nomial reduce + mirrored broadcast:
    2(k−1)·ceil(log_k p) (= Eq. 4's 2·log2 p at k=2)."""
    return 2 * (k - 1) * _levels(p, k)


def crossover_workers(k: int = 2, p_max: int = 1 << 20) -> int:
    """Smallest power-of-two p >= 2 with tree time strictly below PS time
    (S:302-310 enumerates p in {2, 4, 8, ...}; p=1 has no communication)."""
    p = 2
    while p <= p_max:
        if tree_comm_time(1.0, p, 1.0, k) < ps_comm_time(1.0, p, 1.0):
            return p
        p *= 2
    raise ValueError("no crossover below p_max")


def ps_server_bytes(grad_bytes: float, p: int) -> float:
    """Bytes through the server's link for a PS that is also a worker:
    (p−1)·|W| in + (p−1)·|W| out."""
    return 2.0 * (p - 1) * grad_bytes


def allreduce_lower_bound_bytes(grad_bytes: float, p: int) -> float:
    """Per-GPU, per-direction bytes of a bandwidth-optimal allreduce:
    2(p−1)/p·|W| (reduce-scatter + all-gather volume)."""
    return 2.0 * (p - 1) / p * grad_bytes


def single_root_tree_bytes(grad_bytes: float, p: int) -> float:
    """Bytes the root of the paper's single-root binomial tree receives and sends
    (Eq. 4's serialized 2·log2(p)·|W|)."""
    return 2.0 * _levels(p, 2) * grad_bytes
