"""The C ABI used from plain C (examples/c_abi_demo.c, no Python in the loop):
built with gcc against include/firecaffe.h and libfirecaffe.so, run on the GPU,
its results compared bit-exactly with the CPU oracle (-m gpu)."""
import os
import subprocess

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_program_through_the_abi(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA")
    from paper_1511_00175_b200.build import build

    lib = build()
    exe = tmp_path / "c_abi_demo"
    libdir = os.path.dirname(lib)
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "examples", "c_abi_demo.c"), "-L", libdir, "-lfirecaffe",
                           "-L", "/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    out = tmp_path / "out.bin"
    r = subprocess.run([str(exe), str(out)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "c_abi_demo ok" in r.stdout
    p, n = 4, 10007
    a = np.fromfile(out, dtype=np.float32)
    g = a[: p * n].reshape(p, n)
    w0, v0 = a[p * n: p * n + n], a[p * n + n: p * n + 2 * n]
    w_sgd, v_sgd, w_tree = (a[p * n + 2 * n + k * n: p * n + 3 * n + k * n] for k in range(3))
    hp = dict(lr=0.04, mu=0.9, wd=5e-4, batch=1024)
    w_ref, v_ref = oracle.sgd(w0, v0, g[0], **hp)
    assert np.array_equal(w_sgd.view(np.uint32), w_ref.view(np.uint32))
    assert np.array_equal(v_sgd.view(np.uint32), v_ref.view(np.uint32))
    wt_ref, _ = oracle.fused_step(g, w0, v0, **hp)
    assert np.array_equal(w_tree.view(np.uint32), wt_ref.view(np.uint32))
