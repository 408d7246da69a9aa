"""Fused halo push over peer memory (hwg_set_peers).

The stage kernel stores its boundary rows into the neighbour slabs' halo rows
and bumps their arrival counters; the next stage's boundary warps wait on
their own counters.  On one GPU the slabs run on one stream, stage by stage,
so every wait is already satisfied when the kernel starts (no kernel waits
for a concurrently running one); the result must be the single-handle one,
bit for bit.  The two-process test runs the same protocol through CUDA IPC
mappings, the ranks taking turns stage by stage behind a gloo barrier."""
import os

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


def _whole_and_slabs(g, mode, nslabs, stream=None, parts=None):
    from paper_2010_04760_b200.hwgpu import GpuEvolution, SchemeSpec
    from paper_2010_04760_b200.slabs import partition
    n, nt = int(g["nrho"]), int(g["ntheta"])
    spec = SchemeSpec(str(g["scheme"]), mode, float(g["eps"]), float(g["sigma"]))
    whole = GpuEvolution(n, nt, float(g["drho"]), float(g["dtheta"]), int(g["parity"]),
                         g["coef"], g["cotth"], spec)
    whole.set_state(g["u0"])
    slabs = []
    for off, cnt in (parts or partition(n, nslabs)):
        h = GpuEvolution(cnt, nt, float(g["drho"]), float(g["dtheta"]), int(g["parity"]),
                         g["coef"], g["cotth"], spec, rho_offset=off, nrho_global=n)
        u = np.zeros((4, nt + 4, cnt + 8))
        u[:, 2:-2, 4:-4] = g["u0"][:, 2:-2, 4 + off:4 + off + cnt]
        h.set_state(u)
        slabs.append((off, cnt, h))
    return whole, slabs


@pytest.mark.parametrize("case,nslabs", [("kerr09_w5", 2), ("kerr09_w5", 3),
                                         ("extremal_w5_theta34", 2), ("extremal_fd6ko", 3),
                                         ("extremal_w3", 2), ("kerr09_w5_rk104", 3)])
def test_peer_slabs_bit_identical(cuda_ok, case, nslabs):
    from paper_2010_04760_b200.slabs import LocalPeerSlabs
    g = load_golden(case)
    stepper = str(g["stepper"])
    dt = (float(g["dt"][0]), float(g["dt"][1]))
    for mode in ("f64", "mixed"):
        whole, slabs = _whole_and_slabs(g, mode, nslabs)
        whole.launch_steps(stepper, dt, 0, 6)
        ref = whole.get_state()
        ps = LocalPeerSlabs([h for _, _, h in slabs], timeout_s=5.0)
        ps.prime()
        ps.steps(stepper, dt, 0, 6)
        for off, cnt, h in slabs:
            assert h.status() == (False, -1)
            got = h.get_state()
            np.testing.assert_array_equal(got[:, 2:-2, 4:-4], ref[:, 2:-2, 4 + off:4 + off + cnt])
        for _, _, h in slabs:
            h.close()
        whole.close()


@pytest.mark.parametrize("case,parts", [
    ("kerr09_w5", [(0, 24), (24, 48), (72, 24)]),              # uneven: neighbours drift
    ("kerr09_w5", [(0, 16), (16, 16), (32, 32), (64, 32)]),
    ("extremal_w5_theta34", [(0, 40), (40, 80), (120, 40)]),   # 2 theta chunks
    ("extremal_fd6ko", [(0, 20), (20, 44)]),                   # halo 4
    ("kerr09_w5_rk104", [(0, 64), (64, 16), (80, 16)])])       # SSP-RK(10,4)
def test_peer_slabs_concurrent_emulation(cuda_ok, case, parts):
    """The fused halo push under GENUINE concurrency: all slabs
    run in one cooperative launch (hwg_peer_emulate_steps), ordered only by
    the in-kernel pushes and arrival counters, as on separate GPUs.  Repeated
    runs must reproduce the single-handle result bit for bit, no wait may
    time out, and boundary warps must actually have spun on counters bumped
    by running neighbours (hwg_peer_stats; every other run the odd slabs start
    each stage 20 us late, so their neighbours' boundary warps must wait)."""
    from paper_2010_04760_b200.slabs import LocalPeerSlabs
    g = load_golden(case)
    stepper = str(g["stepper"])
    dt = (float(g["dt"][0]), float(g["dt"][1]))
    K = 6
    reps = 100 if case == "kerr09_w5" else 25
    for mode in ("f64", "mixed"):
        whole, slabs = _whole_and_slabs(g, mode, len(parts), parts=parts)
        whole.launch_steps(stepper, dt, 0, K)
        ref = whole.get_state()
        ps = LocalPeerSlabs([h for _, _, h in slabs], timeout_s=5.0)
        spun = 0
        for rep in range(reps):
            for off, cnt, h in slabs:
                u = np.zeros((4, int(g["ntheta"]) + 4, cnt + 8))
                u[:, 2:-2, 4:-4] = g["u0"][:, 2:-2, 4 + off:4 + off + cnt]
                h.set_state(u)
            ps.prime()
            # every other run with the odd slabs late at every stage
            ps.steps_concurrent(stepper, dt, 0, K, skew_ns=20000 if rep % 2 else 0)
            for off, cnt, h in slabs:
                assert h.status() == (False, -1), (rep, off)
                np.testing.assert_array_equal(h.get_state()[:, 2:-2, 4:-4],
                                              ref[:, 2:-2, 4 + off:4 + off + cnt])
        spun = sum(h.peer_stats() for _, _, h in slabs)
        print(case, mode, parts, "spinning waits:", spun)
        assert spun > 0
        for _, _, h in slabs:
            h.close()
        whole.close()


def test_peer_wait_times_out_loudly(cuda_ok):
    """A neighbour that never runs its stage: the waiting boundary warps give
    up after the bounded spin and hwg_status reports the error."""
    from paper_2010_04760_b200.hwgpu import HwgError
    from paper_2010_04760_b200.slabs import LocalPeerSlabs
    g = load_golden("kerr09_w5")
    dt = (float(g["dt"][0]), float(g["dt"][1]))
    whole, slabs = _whole_and_slabs(g, "mixed", 2)
    whole.close()
    ps = LocalPeerSlabs([h for _, _, h in slabs], timeout_s=0.2)
    ps.prime()
    a = slabs[0][2]
    a.launch_stage("ssprk33", 0, dt, 0)  # epoch 0: no wait
    a.launch_stage("ssprk33", 1, dt, 0)  # epoch 1: slab 1 never signalled
    with pytest.raises(HwgError, match="timed out"):
        a.status()


def _ipc_rank(rank, world, port, case, out_dir):
    import torch
    import torch.distributed as dist
    from paper_2010_04760_b200.slabs import PeerSlab
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    g = load_golden(case)
    stepper = str(g["stepper"])
    dt = (float(g["dt"][0]), float(g["dt"][1]))
    whole, slabs = _whole_and_slabs(g, "mixed", world)
    off, cnt, h = slabs[rank]
    for r, (_, _, o) in enumerate(slabs):
        if r != rank:
            o.close()
    ps = PeerSlab(h, rank, world, str(g["scheme"]), timeout_s=5.0)
    ps.prime()
    ns = 3 if stepper == "ssprk33" else 10
    for q in range(4):
        for st in range(ns):
            for r in range(world):  # ranks take turns: waits are satisfied on entry
                if r == rank:
                    h.launch_stage(stepper, st, dt, q)
                    h.synchronize()
                dist.barrier()
    assert h.status() == (False, -1)
    got = h.get_state()[:, 2:-2, 4:-4]
    if rank == 0:
        whole.launch_steps(stepper, dt, 0, 4)
        np.save(os.path.join(out_dir, "whole.npy"), whole.get_state()[:, 2:-2, 4:-4])
    np.save(os.path.join(out_dir, f"slab{rank}.npy"), got)
    dist.barrier()
    dist.destroy_process_group()


def test_peer_slabs_over_cuda_ipc_two_processes(cuda_ok, tmp_path):
    import socket
    import torch.multiprocessing as mp
    from paper_2010_04760_b200.slabs import partition
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    case, world = "kerr09_w5", 2
    mp.start_processes(_ipc_rank, args=(world, port, case, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    ref = np.load(tmp_path / "whole.npy")
    g = load_golden(case)
    for r, (off, cnt) in enumerate(partition(int(g["nrho"]), world)):
        got = np.load(tmp_path / f"slab{r}.npy")
        np.testing.assert_array_equal(got, ref[:, :, off:off + cnt])
