"""Element-partitioned LSRK-45 across GPUs (one process per GPU) with a
per-stage halo exchange of partition-boundary element states.

Per stage, on every rank:
  1. pack the owned elements other ranks hold as ghosts (hw_halo_pack);
  2. start the exchange: NCCL send/recv (torch.distributed, one P2P group per
     stage) straight into the contiguous ghost ranges of q_in;
  3. run the fused stage kernels on the owned *interior* elements (they read
     no ghost) while the exchange is in flight;
  4. wait, form the ghosts' face traces (hw_traces on the ghost subset), run
     the owned *boundary* elements.
The arithmetic per element is the single-GPU kernels' (the same kernels,
on subsets), so partitioned runs reproduce single-GPU results to rounding
(tests/test_gpu_parity.py::test_partitioned_lsrk_loopback).
"""

import numpy as np
import torch

from . import _native as nat
from .dg import Discretization
from .operators import TYPE_ID
from .partition import build_local_parts, partition_elements
from .timeint import LSRK_A, LSRK_B, Stepper

__all__ = ["PartStepper", "NCCLTransport", "LoopbackTransport", "make_parts"]


def make_parts(mesh, nparts, method="xslab", N=3, ranks=None):
    return build_local_parts(mesh, partition_elements(mesh, nparts, method, N=N), ranks=ranks)


class NCCLTransport:
    """Halo exchange over torch.distributed (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def start(self, ps, q):
        d = self.dist
        ops = []
        for peer, per_t in ps.sendbuf.items():
            for t, buf in per_t.items():
                ops.append(d.P2POp(d.isend, buf, peer, group=self.group))
        for peer, per_t in ps.part.recv.items():
            for t, (a, b) in per_t.items():
                ops.append(d.P2POp(d.irecv, q[t][a:b], peer, group=self.group))
        return d.batch_isend_irecv(ops) if ops else []

    def wait(self, handle):
        for w in handle:
            w.wait()


class LoopbackTransport:
    """In-process exchange between PartSteppers sharing one GPU (tests):
    ghost rows are copied from the owning part's current input state."""

    def __init__(self):
        self.steppers = {}

    def start(self, ps, q):
        for peer, per_t in ps.part.recv.items():
            other = self.steppers[peer]
            for t, (a, b) in per_t.items():
                src_idx = other.send_idx[ps.part.rank][t]
                q[t][a:b].copy_(other.S.q[t][src_idx.long()])
        return None

    def wait(self, handle):
        return None


class PartStepper:
    """LSRK-45 on one rank's local part (owned + ghost elements)."""

    def __init__(self, part, N, formulation, state_local, transport, dtype=torch.float64,
                 device=None):
        self.part = part
        self.transport = transport
        self.disc = Discretization(part.mesh, N, formulation, dtype=dtype, device=device)
        d = self.disc
        dev = d.device
        self.S = Stepper(d, state_local, "lsrk")
        empty = torch.zeros(0, dtype=torch.int32, device=dev)

        def lists(kind):
            out = [None] * 4
            for t in d.types:
                lo, hi = {"interior": (0, part.n_interior[t]),
                          "boundary": (part.n_interior[t], part.n_owned[t]),
                          "ghost": (part.n_owned[t], d.n_elems[t])}[kind]
                out[TYPE_ID[t]] = (torch.arange(lo, hi, dtype=torch.int32, device=dev)
                                   if hi > lo else empty)
            return out
        self._keep = [lists("interior"), lists("boundary"), lists("ghost")]
        self.sub_interior, self.sub_boundary, self.sub_ghost = (nat.subset(x) for x in self._keep)
        self.send_idx = {peer: {t: torch.as_tensor(idx, dtype=torch.int32, device=dev)
                                for t, idx in per_t.items()}
                         for peer, per_t in part.send.items()}
        self.sendbuf = {peer: {t: torch.empty((len(idx), 4, d.ops[t].Np), dtype=dtype, device=dev)
                               for t, idx in per_t.items()}
                        for peer, per_t in part.send.items()}
        if isinstance(transport, LoopbackTransport):
            transport.steppers[part.rank] = self
        self.n_dof_owned = sum(part.n_owned[t] * 4 * d.ops[t].Np for t in d.types)

    def launches_per_stage(self):
        """Kernel launches one stage issues (bench gpu_launches): halo packs,
        interior and boundary stage kernels per present type, ghost traces
        per publishing type with ghosts."""
        d, p = self.disc, self.part
        n = sum(len(per_t) for per_t in self.send_idx.values())
        n += sum(1 for t in d.types if p.n_interior[t] > 0)
        n += sum(1 for t in d.types if p.n_owned[t] > p.n_interior[t])
        sem = d.formulation.kind == "SEM"
        pub = ("wedge", "pyramid") if sem else ("hex", "wedge", "pyramid")
        n += sum(1 for t in d.types if t in pub and d.n_elems[t] > p.n_owned[t])
        return n

    def _pack(self, q):
        L, st = nat.lib(), self.disc.stream_ptr()
        dm = self.disc.device_mesh
        for peer, per_t in self.send_idx.items():
            for t, idx in per_t.items():
                nat.check(L.hw_halo_pack(dm.struct, TYPE_ID[t], q[t].data_ptr(), idx.data_ptr(),
                                         idx.numel(), self.sendbuf[peer][t].data_ptr(), st))

    def begin(self):
        """Pack and start the exchange of this stage's input states."""
        self._pack(self.S.q)
        self._handle = self.transport.start(self, self.S.q)

    def finish(self, a, b, h):
        """Interior elements (overlapping the exchange), then the ghosts'
        traces and the boundary elements."""
        S, d = self.S, self.disc
        L, st, dm = nat.lib(), d.stream_ptr(), d.device_mesh
        F = S._f
        handle, self._handle = self._handle, None
        S._stage_traces()
        nat.check(L.hw_lsrk_stage(dm.struct, F(S.q), F(S.q2), F(S.res), a, b, h,
                                  self.sub_interior, st))
        self.transport.wait(handle)
        # ghost traces into the current input trace set
        tin = 1 - S.tr
        nat.check(L.hw_traces(dm.struct, F(S.q), nat.fields(dm.traces[tin]), self.sub_ghost, st))
        nat.check(L.hw_lsrk_stage(dm.struct, F(S.q), F(S.q2), F(S.res), a, b, h,
                                  self.sub_boundary, st))

    def stage(self, a, b, h):
        self.begin()
        self.finish(a, b, h)

    def swap(self):
        self.S.q, self.S.q2 = self.S.q2, self.S.q

    def lsrk_step(self, h):
        for a, b in zip(LSRK_A, LSRK_B):
            self.stage(a, b, h)
            self.swap()

    def owned_state(self):
        return {t: self.S.q[t][:self.part.n_owned[t]] for t in self.disc.types}
