"""Seeded synthetic inputs shared by the tests, smoke() and bench.py.

This module holds NONE of the method's arithmetic (no sums, no SGD): it only
draws random numbers.  Both the oracle side and the CUDA side receive the
tensors it returns, so neither path produces the other's inputs.

Recipe (SURVEY.md §8 d):
  * gradient of rank r: grad_r[i] = sigma_seg(i) · N(0, 1).  The flat vector is
    cut into 64 equal segments (mimicking per-layer blobs) with sigma_seg drawn
    log-uniform in [1e-5, 1e-1] from the base seed (same for every rank, like
    a layer's gradient scale); the normals come from seed + 1000·rank + 1.
    Inputs are per-worker SUMS of ∇W over the worker's sub-batch.
  * weights w ~ N(0, 0.01²) (NiN's 1×1-conv init std); momentum v = 0
    for the first step (reading R10) or N(0, 1e-4²) to exercise the μ·v term.
  * parity-only distributions: "int" (integer-valued, |g| ≤ 2^20 so every
    summation order is exact), "cancel" (±x + small noise across ranks),
    "mixed" (sign·2^U(−30,30)), "subnormal" (values below 2^-126).
"""
from __future__ import annotations

import torch

SEED = 151100175  # arXiv id; fixed base seed for every synthetic input

# BASELINE.json configs: name -> (n_params, default world size, lr, mu, wd, batch)
#   lr/mu/wd/batch from the paper: NiN lr 0.04 @1024, wd 5e-4, mu 0.9
#   (P:358); GoogLeNet lr 0.08, wd 2e-4; AlexNet lr 0.01@256
#   scaled to 0.04@1024, NiN's mu/wd (not stated for AlexNet);
#   VGG-19 not trained in the paper -> NiN's set.
CONFIGS = {
    "tiny": dict(n=1 << 20, p=4, lr=0.04, mu=0.9, wd=5e-4, batch=1024),
    "nin": dict(n=7_600_000, p=8, lr=0.04, mu=0.9, wd=5e-4, batch=1024),
    "googlenet": dict(n=13_250_000, p=8, lr=0.08, mu=0.9, wd=2e-4, batch=1024),
    "alexnet": dict(n=60_965_224, p=8, lr=0.04, mu=0.9, wd=5e-4, batch=1024),
    "vgg19": dict(n=143_667_240, p=8, lr=0.04, mu=0.9, wd=5e-4, batch=1024),
}

N_SEGMENTS = 64


def _gen(device, seed: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def segment_sigmas(seed: int = SEED, n_segments: int = N_SEGMENTS) -> torch.Tensor:
    """Per-segment gradient scale, log-uniform in [1e-5, 1e-1] (CPU, float64)."""
    u = torch.rand(n_segments, generator=_gen("cpu", seed), dtype=torch.float64)
    return torch.pow(10.0, -5.0 + 4.0 * u)


def grad(n: int, rank: int, seed: int = SEED, device="cpu", dist: str = "paper") -> torch.Tensor:
    """Rank `rank`'s fp32 gradient-sum vector of length n."""
    device = torch.device(device)
    g = _gen(device, seed + 1000 * rank + 1)
    if n == 0:
        return torch.empty(0, dtype=torch.float32, device=device)
    if dist == "paper":
        x = torch.randn(n, generator=g, device=device, dtype=torch.float32)
        sig = segment_sigmas(seed).to(torch.float32).to(device)
        seg = (torch.arange(n, device=device, dtype=torch.int64) * N_SEGMENTS) // n
        return x * sig[seg]
    if dist == "int":
        return torch.randint(-(1 << 20), (1 << 20) + 1, (n,), generator=g, device=device).to(torch.float32)
    if dist == "cancel":
        base = torch.randn(n, generator=_gen(device, seed + 7), device=device, dtype=torch.float32)
        sign = 1.0 if rank % 2 == 0 else -1.0
        noise = torch.randn(n, generator=g, device=device, dtype=torch.float32) * 1e-6
        return base * sign + noise
    if dist == "mixed":
        e = torch.randint(-30, 31, (n,), generator=g, device=device).to(torch.float32)
        m = 1.0 + torch.rand(n, generator=g, device=device, dtype=torch.float32)
        s = torch.where(torch.rand(n, generator=g, device=device) < 0.5, -1.0, 1.0)
        return s * m * torch.exp2(e)
    if dist == "subnormal":
        x = torch.randn(n, generator=g, device=device, dtype=torch.float32)
        return x * 1e-39  # mostly below the fp32 normal range (2^-126 ≈ 1.18e-38)
    raise ValueError(f"unknown dist {dist!r}")


def grads(n: int, p: int, seed: int = SEED, device="cpu", dist: str = "paper") -> torch.Tensor:
    """All p ranks' gradients stacked as [p, n] (rank r = row r)."""
    return torch.stack([grad(n, r, seed, device, dist) for r in range(p)]) if p else torch.empty(0, n)


def caffe_blobs(n: int, n_layers: int = 12, seed: int = SEED):
    """A Caffe-like blob table over a flat vector of n params: per layer one
    weight blob (lr_mult 1, decay_mult 1) followed by one bias blob (lr_mult 2,
    decay_mult 0), bias sizes ragged (not multiples of 4).  Returns
    (begins, lr_mults, decay_mults).  For n < 4·n_layers: a single blob."""
    if n < 4 * n_layers:
        return [0], [1.0], [1.0]
    g = _gen("cpu", seed + 17)
    share = torch.rand(n_layers, generator=g, dtype=torch.float64) + 0.2
    sizes = (share / share.sum() * n).floor().to(torch.int64).tolist()
    sizes[-1] += n - sum(sizes)
    begins, lrm, dm, pos = [], [], [], 0
    for s in sizes:
        nb = max(1, min(s // 2, 3 + int(torch.randint(0, 1000, (1,), generator=g))))  # ragged bias
        begins += [pos, pos + s - nb]
        lrm += [1.0, 2.0]
        dm += [1.0, 0.0]
        pos += s
    return begins, lrm, dm


def weights(n: int, seed: int = SEED, device="cpu") -> torch.Tensor:
    """Replicated initial weights, N(0, 0.01²)."""
    return torch.randn(n, generator=_gen(device, seed + 11), device=device, dtype=torch.float32) * 0.01


def momentum(n: int, seed: int = SEED, device="cpu", zero: bool = False) -> torch.Tensor:
    if zero:
        return torch.zeros(n, dtype=torch.float32, device=device)
    return torch.randn(n, generator=_gen(device, seed + 13), device=device, dtype=torch.float32) * 1e-4
