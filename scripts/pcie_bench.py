#!/usr/bin/env python
"""PCIe ceiling for the e2e number: pinned H2D, D2H, and both concurrently on
two streams (30.4 MB each = NiN), plus firecaffe_sgd_step_host at several
pipeline chunk sizes (run once per FC_HOST_MODE / FC_PIPE_CHUNK value)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def t(fn, reps=20):
    torch.cuda.synchronize()
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    return sorted(ms)[reps // 2]


n = 7_600_000
h_in = torch.randn(n).pin_memory()
h_out = torch.empty(n).pin_memory()
d = torch.empty(n, device="cuda")
d2 = torch.randn(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


res = {"h2d_ms": t(lambda: d.copy_(h_in, non_blocking=True)), "d2h_ms": t(lambda: h_out.copy_(d2, non_blocking=True)),
       "both_ms": t(both)}
res = {k: round(v, 4) for k, v in res.items()}
res["h2d_gbs"] = round(4 * n / res["h2d_ms"] / 1e6, 1)
res["d2h_gbs"] = round(4 * n / res["d2h_ms"] / 1e6, 1)
import paper_1511_00175_b200 as fc  # noqa: E402

w, m = torch.randn(n, device="cuda"), torch.zeros(n, device="cuda")
res["sgd_step_host_ms"] = round(t(lambda: fc.firecaffe_sgd_step_host(w, d, m, h_in, h_out, 0.04, 0.9, 5e-4, 1024)), 4)
res["chunk"] = os.environ.get("FC_PIPE_CHUNK", "default")
res["mode"] = os.environ.get("FC_HOST_MODE", "hybrid")
print(json.dumps(res))
