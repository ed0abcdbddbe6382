"""Host-side logic of the N>1 path on CPU (gloo, world_size 2): the IPC-handle
exchange over the process group and the symmetric bump allocator produce the
same offsets on every rank.  No GPU needed."""
import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1511_00175_b200.world import SymmetricLayout, exchange_handles

    mine = bytes([rank]) * 64
    got = exchange_handles(mine, heap_bytes=1 << 30)
    lay = SymmetricLayout(1 << 30, 1 << 20)
    offs = [lay.alloc(n) for n in (4 * 7_600_000, 4 * 7_600_000 + 12, 4 * 5)]
    try:  # a rank with a different heap size is refused on every rank
        exchange_handles(mine, heap_bytes=(1 << 30) + rank)
        refused = False
    except RuntimeError:
        refused = True
    q.put((rank, [g[0] for g in got], offs, refused))
    dist.destroy_process_group()


def test_handle_exchange_and_symmetric_offsets():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [[0, 1], [0, 1]]  # rank-ordered handles on every rank
    assert all(r[3] for r in res)  # mismatched heap sizes refused everywhere
    assert res[0][2] == res[1][2]  # identical offsets -> symmetric buffers
    offs = res[0][2]
    assert all(o % 256 == 0 and o >= (1 << 20) for o in offs)
    assert offs[1] >= offs[0] + 4 * 7_600_000


def test_layout_rejects_overflow():
    from paper_1511_00175_b200.world import SymmetricLayout

    lay = SymmetricLayout(1 << 20, 1 << 16)
    lay.alloc(1000)
    with pytest.raises(MemoryError):
        lay.alloc(1 << 20)
    with pytest.raises(ValueError):
        SymmetricLayout(1 << 16, 1 << 16)
