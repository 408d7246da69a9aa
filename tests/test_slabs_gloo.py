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


def _worker(rank, world, port, case, steps, q):
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
    DistSlab(b, rank, world, str(g["scheme"])).steps("ssprk33", float(g["dt"][0]), 0, steps)
    q.put((rank, off, b.interior()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_slabs_match_single_domain(world):
    from conftest import load_golden
    from helpers import oracle_from_golden
    case, steps = "kerr09_w5", 4
    g = load_golden(case)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, steps, q))
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
