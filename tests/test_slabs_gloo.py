"""CPU tests of the radial-slab runtime (paper_2010_04760_b200/slabs.py) under
torch.distributed gloo, world_size 2 and 3: the slab decomposition with
per-stage halo exchange reproduces the single-domain oracle evolution
bitwise (the multi-rank analogue of the reference's worker-count
bit-identity, proj/tests/test_evolve.cpp:363-395)."""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, case, steps, q, overlap=False):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist
    from conftest import load_golden
    from paper_2010_04760_b200.slabs import DistSlab, partition
    from slab_cpu_backend import CpuSlab
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    g = load_golden(case)
    off, cnt = partition(int(g["nrho"]), world)[rank]
    b = CpuSlab(g, off, cnt)
    b.set_interior(g["u0"][:, 2:-2, 4 + off:4 + off + cnt])
    DistSlab(b, rank, world, str(g["scheme"]), overlap=overlap).steps(
        "ssprk33", float(g["dt"][0]), 0, steps)
    q.put((rank, off, b.interior()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,overlap", [(2, False), (3, False), (2, True), (3, True)])
def test_gloo_slabs_match_single_domain(world, overlap):
    from conftest import load_golden
    from helpers import oracle_from_golden
    case, steps = "kerr09_w5", 4
    g = load_golden(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, steps, q, overlap))
             for r in range(world)]
    for p in procs:
        p.start()
    parts = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    orc = oracle_from_golden(g, "f64")
    ref, _ = orc.advance(g["u0"], float(g["dt"][0]), 0, steps)
    ref = ref[:, 2:-2, 4:-4]
    for rank, off, u in parts:
        np.testing.assert_array_equal(u, ref[:, :, off:off + u.shape[2]])


def test_partition_balanced():
    from paper_2010_04760_b200.slabs import partition
    for n, w in ((65536, 8), (1000, 3), (17, 4)):
        p = partition(n, w)
        assert sum(c for _, c in p) == n
        assert max(c for _, c in p) - min(c for _, c in p) <= 1
        assert all(p[i][0] + p[i][1] == p[i + 1][0] for i in range(w - 1))


class _MockPeerBackend:
    """Records what PeerSlab hands to hwg_set_peers (no GPU)."""

    def __init__(self, rank, fail=False):
        self.rank, self.fail, self.calls = rank, fail, []

    def peer_export(self):
        return f"desc-{self.rank}".encode()

    def set_peers(self, lower, upper, ipc=False, timeout_s=10.0):
        self.calls.append((lower, upper, ipc))
        if self.fail:
            raise RuntimeError("cudaIpcOpenMemHandle: not permitted")


def _peer_worker(rank, world, port, fail_rank, q):
    sys.path.insert(0, HERE)
    sys.path.insert(0, os.path.dirname(HERE))
    import torch.distributed as dist
    from paper_2010_04760_b200.slabs import PeerSlab
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    b = _MockPeerBackend(rank, fail=rank == fail_rank)
    ps = PeerSlab(b, rank, world, "weno5")
    q.put((rank, b.calls, None if ps.error is None else str(ps.error)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,fail_rank", [(3, -1), (2, 1)])
def test_peer_slab_setup_wires_neighbours(world, fail_rank):
    """PeerSlab's collective setup (descriptor all-gather over the process
    group): rank r connects desc r-1 below and r+1 above over IPC, the ends
    have no neighbour, and a rank whose mapping fails still reaches the
    barrier and reports the error instead of hanging the others."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, fail_rank, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict((r, (c, e)) for r, c, e in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        calls, err = got[r]
        lower = f"desc-{r - 1}".encode() if r > 0 else None
        upper = f"desc-{r + 1}".encode() if r < world - 1 else None
        assert calls == [(lower, upper, True)]
        assert (err is not None) == (r == fail_rank)
