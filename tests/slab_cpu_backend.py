"""TEST INFRASTRUCTURE: a CPU stand-in for one radial-slab GpuEvolution handle,
so the multi-rank slab logic (paper_2010_04760_b200/slabs.py) runs under
torch.distributed gloo on CPU.

It mirrors the handle's surface used by slabs.DistSlab (nrho, stage_input,
register_view, launch_stage) and its register rotation (hwg_solver.cu
do_stage) with torch CPU tensors in the device row layout, and evaluates each
stage with the oracle C restatement on the slab extended by its halo rows.
"""
from __future__ import annotations

import numpy as np
import torch

from oracle import OracleSolver

HALO = 4


def to_rows(u_interior: np.ndarray, nchunks: int) -> np.ndarray:
    """(4, nt, n) interior -> (n, nchunks*64*2) device row layout."""
    _, nt, n = u_interior.shape
    out = np.zeros((n, nchunks, 2, 32, 2))
    for c in range(4):
        plane, comp = divmod(c, 2)
        for k in range(nt):
            out[:, k // 32, plane, k % 32, comp] = u_interior[c, k, :]
    return out.reshape(n, -1)


def from_rows(rows: np.ndarray, nt: int) -> np.ndarray:
    n = rows.shape[0]
    v = rows.reshape(n, -1, 2, 32, 2)
    out = np.zeros((4, nt, n))
    for c in range(4):
        plane, comp = divmod(c, 2)
        for k in range(nt):
            out[c, k, :] = v[:, k // 32, plane, k % 32, comp]
    return out


class CpuSlab:
    def __init__(self, g: dict, off: int, cnt: int, mode: str = "f64"):
        self.g, self.off, self.nrho = g, off, cnt
        self.nt = int(g["ntheta"])
        self.nglob = int(g["nrho"])
        self.nchunks = (self.nt + 31) // 32
        self.mode = mode
        self.row = self.nchunks * 64 * 2
        self.regs = [torch.zeros(cnt + 2 * HALO, self.row, dtype=torch.float64) for _ in range(3)]
        self.cur, self.scr1, self.scr2 = 0, 1, 2

    def set_interior(self, u_interior: np.ndarray):
        self.regs[self.cur][HALO:HALO + self.nrho] = torch.from_numpy(
            to_rows(u_interior, self.nchunks))

    def interior(self) -> np.ndarray:
        return from_rows(self.regs[self.cur][HALO:HALO + self.nrho].numpy(), self.nt)

    def register_view(self, reg: int):
        return self.regs[reg]

    def stage_input(self, stepper: str, stage: int) -> int:
        assert stepper == "ssprk33"
        return (self.cur, self.scr1, self.scr2)[stage]

    def _rhs(self, reg: int, poison_halo: bool = False) -> np.ndarray:
        """F of the slab interior from register `reg` (halo rows valid, or
        replaced by NaN in a copy when they may still be in flight)."""
        g = self.g
        lo = 0 if self.off == 0 else 3
        hi = 0 if self.off + self.nrho == self.nglob else 3
        r0, r1 = self.off - lo, self.off + self.nrho + hi
        ext = from_rows(self.regs[reg][HALO - lo:HALO + self.nrho + hi].numpy(), self.nt)
        if poison_halo:
            if lo:
                ext[:, :, :lo] = np.nan
            if hi:
                ext[:, :, -hi:] = np.nan
        m = r1 - r0
        coef = g["coef"].reshape(9, self.nt, self.nglob)[:, :, r0:r1]
        orc = OracleSolver(m, self.nt, float(g["drho"]), float(g["dtheta"]), int(g["parity"]),
                           np.ascontiguousarray(coef), g["cotth"], str(g["scheme"]), self.mode,
                           float(g["eps"]), float(g["sigma"]))
        u = np.zeros((4, self.nt + 4, m + 8))
        u[:, 2:-2, 4:-4] = ext
        _, du = orc.rhs(u)
        return du[:, 2:-2, 4 + lo:4 + lo + self.nrho]

    def launch_stage(self, stepper: str, stage: int, dt, step: int):
        self.launch_stage_rows(stepper, stage, dt, step, 0, self.nrho, True, True)

    def launch_stage_rows(self, stepper: str, stage: int, dt, step: int, row_lo: int,
                          row_hi: int, first: bool, last: bool):
        """hwg_launch_stage_rows: write output rows [row_lo, row_hi) only;
        rotate the registers on the stage's last part.  A part launched
        while its halo rows are still in flight must not depend on them: the
        halo rows are replaced by NaN (in the copy the stage reads) unless the
        part touches a slab end (then the exchange has completed,
        DistSlab.step)."""
        dt = dt[0] if isinstance(dt, tuple) else dt
        x = self.stage_input(stepper, stage)
        self._stage(stepper, stage, dt, x, row_lo, row_hi,
                    poison=row_lo >= 3 and row_hi <= self.nrho - 3)
        if last and stage == 2:
            self.cur, self.scr1 = self.scr1, self.cur

    def _stage(self, stepper, stage, dt, x, row_lo, row_hi, poison=False):
        # ssprk33_step (proj/include/hweno/timestep.hpp:54-71), interior only
        f = self._rhs(x, poison)
        X = from_rows(self.regs[x][HALO:HALO + self.nrho].numpy(), self.nt)
        U = from_rows(self.regs[self.cur][HALO:HALO + self.nrho].numpy(), self.nt)
        if stage == 0:
            out, dst = X + dt * f, self.scr1
        elif stage == 1:
            out, dst = 0.75 * U + 0.25 * (X + dt * f), self.scr2
        else:
            out, dst = (1.0 / 3.0) * U + (2.0 / 3.0) * (X + dt * f), self.scr1
        rows = torch.from_numpy(to_rows(out, self.nchunks))
        self.regs[dst][HALO + row_lo:HALO + row_hi] = rows[row_lo:row_hi]
