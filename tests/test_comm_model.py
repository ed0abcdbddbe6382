"""The product's planning model (paper_1511_00175_b200.comm_model) vs the
oracle's independent Eq. 3/4 (oracle/comm_model.py), and the calibration fit."""
import pytest

from oracle import comm_model as ocm
from paper_1511_00175_b200 import comm_model as pcm


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8, 16, 128])
@pytest.mark.parametrize("k", [2, 3, 4])
def test_closed_forms_match_oracle(p, k):
    W, bw = 30e6, 1e9
    assert pcm.eq3_param_server(W, p, bw) == pytest.approx(ocm.ps_comm_time(W, p, bw), rel=1e-15)
    assert pcm.eq4_reduction_tree(W, p, bw, k) == pytest.approx(ocm.tree_comm_time(W, p, bw, k), rel=1e-15)


def test_schedule_bytes():
    W = 1.0
    assert pcm.schedule_bytes("flat", W, 8) == pytest.approx(ocm.allreduce_lower_bound_bytes(W, 8))
    assert pcm.schedule_bytes("forest", W, 4) == pytest.approx(1.5)
    assert pcm.schedule_bytes("ps", W, 8) == pytest.approx(ocm.ps_server_bytes(W, 8) / 2)  # per direction
    assert pcm.schedule_bytes("single_root", W, 8) == pytest.approx(ocm.single_root_tree_bytes(W, 8) / 2)
    assert pcm.schedule_bytes("flat", W, 1) == 0.0


def test_calibration_recovers_parameters():
    bw, t0 = 680e9, 22e-6
    pts = [(s, 4.0 * n, p, t0 + pcm.schedule_bytes(s, 4.0 * n, p) / bw)
           for s in ("flat", "ps") for n in (7_600_000, 60_965_224) for p in (2, 4)]
    c = pcm.calibrate(pts)
    assert c.bw == pytest.approx(bw, rel=1e-9)
    assert c.t0 == pytest.approx(t0, rel=1e-6)
    assert c.predict("flat", 4.0 * 7_600_000, 8) == pytest.approx(t0 + 1.75 * 30.4e6 / bw)
