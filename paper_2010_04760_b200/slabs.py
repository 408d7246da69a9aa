"""Radial-slab domain decomposition across GPUs.

The grid is cut into contiguous rho slabs (theta unsplit); each rank owns one
slab in one GpuEvolution handle.  Before every RK stage the stage's stencil
input register exchanges its boundary rows with both neighbours — the only
data-path communication of the hot path (the reference has none: it is a
single shared-memory process, proj/include/hweno/parallel.hpp).  Halo rows
are plain copies, and the stage kernel computes every interface with the
same instruction sequence wherever it sits, so the result is bitwise the
single-GPU one.

Transports:
  * PeerSlab   — the B200 path: no per-stage collective at all.  Every stage
                 kernel stores its boundary rows straight into the
                 neighbours' halo rows over NVLink (CUDA IPC mappings) and
                 bumps their arrival counters; the next stage's boundary
                 warps wait on them (hwg_set_peers).  One process per GPU.
  * LocalPeerSlabs — the same kernels with several slabs in one process
                 (same-device pointers; on one GPU the slabs' stages are
                 launched in order, so every wait is already satisfied);
  * DistSlab   — torch.distributed point-to-point (NCCL over NVLink on GPUs,
                 gloo on CPU), one process per GPU: the collective baseline.
                 With overlap=True the exchange is posted,
                 the interior rows [h, n-h) — which need no halo — run while
                 it is in flight, then the two h-row boundary strips;
  * LocalSlabs — several handles in one process, halos copied with
                 stream-ordered device copies (bit-identity checks on one GPU).
"""
from __future__ import annotations

HALO_ROWS = {"weno5": 3, "weno3": 2, "fd6ko": 4}
BUF_HALO = 4  # halo rows allocated per side in every register


def partition(nrho_global: int, world: int):
    """Balanced contiguous partition [(offset, count)] (WorkerPool::slice rule,
    proj/include/hweno/parallel.hpp:51-55)."""
    out = []
    for r in range(world):
        b = nrho_global * r // world
        e = nrho_global * (r + 1) // world
        out.append((b, e - b))
    return out


def halo_views(backend, reg: int, h: int):
    """(send_left, recv_left, send_right, recv_right) row views of register
    `reg` (a row is contiguous, so each is one contiguous message)."""
    v = backend.register_view(reg)
    n = backend.nrho
    H = BUF_HALO
    return v[H:H + h], v[H - h:H], v[H + n - h:H + n], v[H + n:H + n + h]


class DistSlab:
    """One rank's slab; halos through torch.distributed P2P."""

    def __init__(self, backend, rank: int, world: int, scheme: str = "weno5", group=None,
                 overlap: bool = False):
        self.b = backend
        self.rank, self.world = rank, world
        self.left = rank - 1 if rank > 0 else None
        self.right = rank + 1 if rank < world - 1 else None
        self.h = HALO_ROWS[scheme]
        self.group = group
        self._copy_back = []
        # interior / strips need >= 2 rows each (hwg_launch_stage_rows)
        self.overlap = (overlap and world > 1 and hasattr(backend, "launch_stage_rows")
                        and backend.nrho >= 2 * self.h + 2)

    def _staged(self, t) -> bool:
        """Device rows over a host-only backend (gloo): exchange through host
        copies (NCCL moves device rows directly)."""
        import torch.distributed as dist
        return t.is_cuda and dist.get_backend(self.group) != "nccl"

    def post(self, reg: int):
        """Post the halo exchange of register `reg`; returns the requests
        (pass them to wait())."""
        import torch.distributed as dist
        self._copy_back = []
        if self.world == 1:
            return []
        sl, rl, sr, rr = halo_views(self.b, reg, self.h)
        if self._staged(sl):
            self.b.synchronize()  # the stage that wrote the rows is done
            host = lambda t: t.cpu()  # noqa: E731
            rl_h, rr_h = rl.cpu(), rr.cpu()
            self._copy_back = [(rl, rl_h), (rr, rr_h)]
            sl, sr, rl, rr = host(sl), host(sr), rl_h, rr_h
        ops = []
        if self.left is not None:
            ops.append(dist.P2POp(dist.isend, sl, self.left, self.group))
            ops.append(dist.P2POp(dist.irecv, rl, self.left, self.group))
        if self.right is not None:
            ops.append(dist.P2POp(dist.isend, sr, self.right, self.group))
            ops.append(dist.P2POp(dist.irecv, rr, self.right, self.group))
        return dist.batch_isend_irecv(ops)

    def wait(self, reqs):
        for req in reqs:
            req.wait()
        if self._copy_back:
            import torch
            for dev, hst in self._copy_back:
                dev.copy_(hst)
            torch.cuda.synchronize()  # rows in place before the handle's next launch
            self._copy_back = []

    def exchange(self, reg: int):
        self.wait(self.post(reg))

    def step(self, stepper: str, dt, step: int):
        ns = 3 if stepper == "ssprk33" else 10
        n, h = self.b.nrho, self.h
        for st in range(ns):
            reqs = self.post(self.b.stage_input(stepper, st))
            if not self.overlap:
                self.wait(reqs)
                self.b.launch_stage(stepper, st, dt, step)
                continue
            # interior rows while the halo rows are in flight (NCCL: the
            # kernel is queued behind nothing but the previous stage; wait()
            # then orders the strips after the exchange on the device)
            self.b.launch_stage_rows(stepper, st, dt, step, h, n - h, True, False)
            self.wait(reqs)
            self.b.launch_stage_rows(stepper, st, dt, step, 0, h, False, False)
            self.b.launch_stage_rows(stepper, st, dt, step, n - h, n, False, True)

    def steps(self, stepper: str, dt, step_begin: int, nsteps: int):
        for q in range(nsteps):
            self.step(stepper, dt, step_begin + q)


class PeerSlab:
    """One rank's slab with the fused halo push (hwg_set_peers over CUDA IPC).
    Setup is collective over `group` (descriptor all-gather + barriers); the
    stage loop itself issues no collective."""

    def __init__(self, backend, rank: int, world: int, scheme: str = "weno5", group=None,
                 timeout_s: float = 10.0):
        import torch.distributed as dist
        self.b = backend
        self.rank, self.world = rank, world
        self.group = group
        mine = backend.peer_export()
        descs = [None] * world
        dist.all_gather_object(descs, mine, group=group)
        lower = descs[rank - 1] if rank > 0 else None
        upper = descs[rank + 1] if rank < world - 1 else None
        self.error = None
        try:
            backend.set_peers(lower, upper, ipc=True, timeout_s=timeout_s)
        except Exception as e:  # e.g. CUDA IPC not permitted: every rank still reaches the barrier
            self.error = e
        dist.barrier(group=group)

    def prime(self):
        """Initial halos of the current register (after set_state on every rank)."""
        import torch.distributed as dist
        dist.barrier(group=self.group)
        self.b.peer_prime()
        dist.barrier(group=self.group)

    def exchange(self, reg: int):  # the kernels carry the halos
        return

    def step(self, stepper: str, dt, step: int):
        ns = 3 if stepper == "ssprk33" else 10
        for st in range(ns):
            self.b.launch_stage(stepper, st, dt, step)

    def steps(self, stepper: str, dt, step_begin: int, nsteps: int):
        self.b.launch_steps(stepper, dt, step_begin, nsteps)


class LocalPeerSlabs:
    """Fused-halo slabs in one process on ONE device: all slabs launch on one
    stream, slab by slab and stage by stage, so a stage kernel only ever waits
    for kernels that already finished (never for a concurrently running one)."""

    def __init__(self, backends, timeout_s: float = 10.0):
        import torch
        self.bs = list(backends)
        self.stream = torch.cuda.Stream()
        for b in self.bs:
            b.set_stream(self.stream.cuda_stream)
        d = [b.peer_export() for b in self.bs]
        for i, b in enumerate(self.bs):
            b.set_peers(d[i - 1] if i > 0 else None, d[i + 1] if i + 1 < len(d) else None,
                        ipc=False, timeout_s=timeout_s)

    def prime(self):
        for b in self.bs:
            b.synchronize()
        for b in self.bs:
            b.peer_prime()

    def step(self, stepper: str, dt, step: int):
        ns = 3 if stepper == "ssprk33" else 10
        for st in range(ns):
            for b in self.bs:
                b.launch_stage(stepper, st, dt, step)

    def steps(self, stepper: str, dt, step_begin: int, nsteps: int):
        for q in range(nsteps):
            self.step(stepper, dt, step_begin + q)

    def steps_concurrent(self, stepper: str, dt, step_begin: int, nsteps: int, skew_ns: int = 0):
        """All slabs' stages in ONE cooperative launch (hwg_peer_emulate_steps):
        the slabs run concurrently and are ordered only by the fused push's
        counters, as on separate GPUs — boundary warps really wait."""
        from .hwgpu import peer_emulate_steps
        peer_emulate_steps(self.bs, stepper, dt, step_begin, nsteps, skew_ns)


class LocalSlabs:
    """Several slab handles in one process (one GPU or CPU backends).  With
    overlap=True every stage runs as DistSlab's overlapped sequence: interior
    parts, then the halo copies (so the interior parts see the previous
    stage's halo rows — a dependence on them would show), then the strips."""

    def __init__(self, backends, scheme: str = "weno5", overlap: bool = False):
        self.bs = list(backends)
        self.h = HALO_ROWS[scheme]
        self.overlap = overlap

    def exchange(self, regs):
        views = [halo_views(b, r, self.h) for b, r in zip(self.bs, regs)]
        for i in range(len(self.bs) - 1):
            _, _, sr, rr = views[i]
            sl, rl, _, _ = views[i + 1]
            rl.copy_(sr)   # right neighbour's left halo <- my last rows
            rr.copy_(sl)   # my right halo <- right neighbour's first rows

    def step(self, stepper: str, dt, step: int):
        ns = 3 if stepper == "ssprk33" else 10
        h = self.h
        for st in range(ns):
            regs = [b.stage_input(stepper, st) for b in self.bs]
            if self.overlap:
                for b in self.bs:
                    b.launch_stage_rows(stepper, st, dt, step, h, b.nrho - h, True, False)
            self.exchange(regs)
            for b in self.bs:
                if self.overlap:
                    b.launch_stage_rows(stepper, st, dt, step, 0, h, False, False)
                    b.launch_stage_rows(stepper, st, dt, step, b.nrho - h, b.nrho, False, True)
                else:
                    b.launch_stage(stepper, st, dt, step)

    def steps(self, stepper: str, dt, step_begin: int, nsteps: int):
        for q in range(nsteps):
            self.step(stepper, dt, step_begin + q)
