"""Element-partitioned LSRK-45 across GPUs (one process per GPU) with a
per-stage face-level halo exchange.

A ghost element is read by my boundary elements only through the face it
shares with them: its face nodes (tet, SEM hex: selection traces of the
state) or its published face traces (wedge, pyramid, GL hex).  So only
those face values travel (hex N=4: 4 x 25 values per cut face instead of
the 4 x 125 of a whole element state).  Per stage, on every rank:
  1. gather the shared-face values of my owned elements the peers touch
     (hw_halo_gather: face nodes of q_in, or my input-trace rows);
  2. start the exchange: NCCL send/recv (torch.distributed, one batched P2P
     group per stage) into per-peer receive buffers;
  3. run the fused stage kernels on the owned *interior* elements (they read
     no ghost) while the exchange is in flight;
  4. wait, scatter the received face values into the ghosts' state rows /
     input-trace rows (hw_halo_scatter), run the owned *boundary* elements.
The arithmetic per element is the single-GPU kernels' (the same kernels,
on subsets), so partitioned runs reproduce single-GPU results to rounding
(tests/test_gpu_parity.py::test_partitioned_lsrk_loopback).
"""

import functools

import numpy as np

import torch

from . import _native as nat
from .dg import Discretization
from .operators import TYPE_ID
from .partition import build_local_parts, partition_elements
from .timeint import LSRK_A, LSRK_B, Stepper

__all__ = ["PartStepper", "PartMRAB", "NCCLTransport", "LoopbackTransport", "make_parts"]


def make_parts(mesh, nparts, method="xslab", N=3, ranks=None):
    return build_local_parts(mesh, partition_elements(mesh, nparts, method, N=N), ranks=ranks)


class NCCLTransport:
    """Halo exchange over torch.distributed (NCCL on GPUs, gloo on CPU):
    ``ps.send_buffers()`` / ``ps.recv_buffers(q)`` list (peer, tensor) in
    the canonical (peer, element type) order both sides derive from the
    global partition, so the batched P2P operations pair up."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group

    def start(self, ps, q):
        d = self.dist
        ops = [d.P2POp(d.isend, buf, peer, group=self.group) for peer, buf in ps.send_buffers()]
        ops += [d.P2POp(d.irecv, buf, peer, group=self.group)
                for peer, buf in ps.recv_buffers(q)]
        return d.batch_isend_irecv(ops) if ops else []

    def wait(self, handle):
        for w in handle:
            w.wait()


class LoopbackTransport:
    """In-process exchange between the parts of one partition sharing one
    GPU (tests): each receiver pulls its halo from the owning part."""

    def __init__(self):
        self.steppers = {}

    def start(self, ps, q):
        for peer in ps.part.recv:
            ps.receive_from(self.steppers[peer], q)
        return None

    def wait(self, handle):
        return None


def face_halo_offsets(t, dops, N, sem):
    """Per face of type t: (offsets of the face's values within one element
    row of the halo source, field stride kind).  Tet and SEM hex faces are
    read from the state (face nodes), the publishing types from their trace
    rows (device face-point order)."""
    fo = np.asarray(dops["face_offsets"])
    nf = len(fo) - 1
    if t == "tet":
        nfn = len(dops["face_nodes"]) // 4
        fn = np.asarray(dops["face_nodes"]).reshape(4, nfn)
        return [fn[f].astype(np.int64) for f in range(4)], "state"
    if t == "hex" and sem:
        tab = np.asarray(dops["face_tab"]).reshape(-1, 3)
        return [(tab[fo[f]:fo[f + 1], 0] + np.where(tab[fo[f]:fo[f + 1], 2] != 0, N, 0)
                 * tab[fo[f]:fo[f + 1], 1]).astype(np.int64) for f in range(nf)], "state"
    return [np.arange(fo[f], fo[f + 1], dtype=np.int64) for f in range(nf)], "trace"


def flat_face_offsets(pairs, local, row):
    """Flat field-0 offsets of the (element, face) pairs' values: element *
    row + the face's offsets within the row (row = 4 * Np or 4 * Nfp)."""
    if len(pairs) == 0:
        return np.zeros(0, dtype=np.int64)
    return np.concatenate([int(k) * row + local[int(f)] for k, f in pairs])


def _split_corrections(dm, part):
    """The face-correction rows (device.wedge_face_corrections) of a rank's
    local mesh split by the wedge they read: (owned wedge, ghost wedge).  A
    row of an interior element always reads an owned wedge."""
    nfp_w = dm.pack["types"]["wedge"]["nfp"]
    n_own = part.n_owned["wedge"]
    own_rows, ghost_rows = {}, {}
    for t, c in dm.corr.items():
        wk = c["idata"][:, 2].long() // (4 * nfp_w)       # wedge of the row's first face node
        for dst, m in ((own_rows, wk < n_own), (ghost_rows, wk >= n_own)):
            n = int(m.sum())
            if n:
                dst[t] = {**c, "n": n, "idata": c["idata"][m].contiguous(),
                          "fdata": c["fdata"][m].contiguous()}
    return own_rows, ghost_rows


class PartStepper:
    """LSRK-45 on one rank's local part (owned + ghost elements)."""

    def __init__(self, part, N, formulation, state_local, transport, dtype=torch.float64,
                 device=None):
        self.part = part
        self.transport = transport
        self.disc = Discretization(part.mesh, N, formulation, dtype=dtype, device=device)
        d = self.disc
        dev = d.device
        # tets / pyramids across non-affine wedge triangles: correction rows
        # of owned wedges before the interior launch, of ghost wedges after
        # the halo (their traces) has arrived
        self.corr_rows = _split_corrections(d.device_mesh, part) if d.device_mesh.corr else None
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
        # face-level halo: flat offsets of the shared faces' values in the
        # halo source (state rows or trace rows) on both sides
        pack = dm_pack = d.device_mesh.pack
        sem = d.formulation.kind == "SEM"
        self.kind, self.row, self.fstride = {}, {}, {}
        local = {}
        for t in d.types:
            local[t], self.kind[t] = face_halo_offsets(t, dm_pack["types"][t]["dops"], N, sem)
            nfp = pack["types"][t]["nfp"]
            Np = d.ops[t].Np
            self.fstride[t] = Np if self.kind[t] == "state" else nfp
            self.row[t] = 4 * self.fstride[t]
        as_dev = lambda a: torch.as_tensor(a, dtype=torch.int64, device=dev)
        self.send_off = {peer: {t: as_dev(flat_face_offsets(pr, local[t], self.row[t]))
                                for t, pr in per_t.items()}
                         for peer, per_t in part.send_faces.items()}
        self.recv_off = {peer: {t: as_dev(flat_face_offsets(pr, local[t], self.row[t]))
                                for t, pr in per_t.items()}
                         for peer, per_t in part.recv_faces.items()}
        self.sendbuf = {peer: {t: torch.empty(4 * o.numel(), dtype=dtype, device=dev)
                               for t, o in per_t.items()}
                        for peer, per_t in self.send_off.items()}
        self.recvbuf = {peer: {t: torch.empty(4 * o.numel(), dtype=dtype, device=dev)
                               for t, o in per_t.items()}
                        for peer, per_t in self.recv_off.items()}
        if isinstance(transport, LoopbackTransport):
            transport.steppers[part.rank] = self
        self.n_dof_owned = sum(part.n_owned[t] * 4 * d.ops[t].Np for t in d.types)
        self.halo_bytes = sum(b.numel() * b.element_size()
                              for per_t in self.recvbuf.values() for b in per_t.values())

    def _source(self, t, tr_set):
        return (self.S.q[t] if self.kind[t] == "state"
                else self.disc.device_mesh.traces[tr_set][TYPE_ID[t]])

    def send_buffers(self):
        return [(peer, self.sendbuf[peer][t]) for peer in sorted(self.sendbuf)
                for t in self.disc.types if t in self.sendbuf[peer]]

    def recv_buffers(self, q):
        return [(peer, self.recvbuf[peer][t]) for peer in sorted(self.recvbuf)
                for t in self.disc.types if t in self.recvbuf[peer]]

    def receive_from(self, other, q):
        """Loopback: the owning part gathers my halo from its current input."""
        other._pack(only=self.part.rank)
        for t, buf in self.recvbuf[other.part.rank].items():
            buf.copy_(other.sendbuf[self.part.rank][t])

    def launches_per_stage(self):
        """Kernel launches one stage issues (bench gpu_launches): halo
        gathers and scatters, interior and boundary stage kernels per
        present type."""
        d, p = self.disc, self.part
        n = sum(len(per_t) for per_t in self.send_off.values())
        n += sum(len(per_t) for per_t in self.recv_off.values())
        n += sum(1 for t in d.types if p.n_interior[t] > 0)
        n += sum(1 for t in d.types if p.n_owned[t] > p.n_interior[t])
        return n

    def _pack(self, only=None):
        """Gather the shared-face values of this stage's input (state q_in,
        input trace set) for the peers (only: one peer)."""
        L, st = nat.lib(), self.disc.stream_ptr()
        dm = self.disc.device_mesh
        for peer, per_t in self.send_off.items():
            if only is not None and peer != only:
                continue
            for t, off in per_t.items():
                src = self._source(t, self.S.tr)
                nat.check(L.hw_halo_gather(dm.struct, src.data_ptr(), self.fstride[t],
                                           off.data_ptr(), off.numel(),
                                           self.sendbuf[peer][t].data_ptr(), st))

    def begin(self):
        """Gather and start the exchange of this stage's shared-face values."""
        if not isinstance(self.transport, LoopbackTransport):
            self._pack()
        self._handle = self.transport.start(self, self.S.q)

    def finish(self, a, b, h):
        """Interior elements (overlapping the exchange), then the received
        face values into the ghosts and the boundary elements."""
        S, d = self.S, self.disc
        L, st, dm = nat.lib(), d.stream_ptr(), d.device_mesh
        F = S._f
        handle, self._handle = self._handle, None
        tin = S.tr                      # input trace set of this stage
        S._stage_traces()
        if self.corr_rows is not None:
            d.apply_corrections(rows=self.corr_rows[0])
        nat.check(L.hw_lsrk_stage(dm.struct, F(S.q), F(S.q2), F(S.res), a, b, h,
                                  self.sub_interior, st))
        self.transport.wait(handle)
        for peer, per_t in self.recv_off.items():
            for t, off in per_t.items():
                dst = self._source(t, tin)
                nat.check(L.hw_halo_scatter(dm.struct, self.recvbuf[peer][t].data_ptr(),
                                            self.fstride[t], off.data_ptr(), off.numel(),
                                            dst.data_ptr(), st))
        if self.corr_rows is not None and self.corr_rows[1]:
            d.apply_corrections(rows=self.corr_rows[1], zero=False)
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


@functools.lru_cache(maxsize=None)
def _ab_coeffs(nh):
    """AB coefficients of a full step, padded to 3 (hybridwave/timeint.py:21-38)."""
    from .timeint import ab_coefficients
    return tuple(float(x) for x in ab_coefficients(nh)) + (0.0,) * (3 - nh)


@functools.lru_cache(maxsize=None)
def _dense_coeffs(nh, frac, period):
    """Dense-output coefficients c(theta) - c(1), theta = frac / period
    (hybridwave/timeint.py:144-173), padded to 3."""
    from .timeint import ab_coefficients
    c = ab_coefficients(nh, frac / period) - ab_coefficients(nh, 1.0)
    return tuple(float(x) for x in c) + (0.0,) * (3 - nh)


class PartMRAB:
    """Multi-rate AB3 (timeint.MRABDriver's tick pattern) on one rank's local
    part.  Each tick: dense-output (effective) state of the owned elements
    the tick reads plus the partition-boundary elements the peers read,
    exchange of the boundary elements' effective state into the peers'
    ghost rows, traces of the elements read, fused RHS + AB3 update of the
    owned stepping elements.  Ghost elements never step; their history lives
    on the owning rank, so every value a rank consumes equals the single-GPU
    run's (tests/test_gpu_parity.py::test_partitioned_mrab_loopback)."""

    def __init__(self, part, N, formulation, state_local, levels_local, n_levels, transport,
                 dtype=torch.float64, device=None):
        from .timeint import ab_coefficients   # noqa: F401 (used in tick)
        self.part = part
        self.transport = transport
        self.disc = d = Discretization(part.mesh, N, formulation, dtype=dtype, device=device)
        dev = d.device
        self.L = L = int(n_levels)
        self.levels = {t: np.asarray(levels_local[t]) for t in d.types}
        self.q = d.to_device(state_local)
        self.eff = d.empty_state()
        self.ring = [d.zeros_state() for _ in range(3)]
        self._fcache = {}
        self.n_hist = np.zeros(L + 1, dtype=int)
        self.steps = np.zeros(L + 1, dtype=int)
        self.send_idx = {peer: {t: torch.as_tensor(idx, dtype=torch.int32, device=dev)
                                for t, idx in per_t.items()}
                         for peer, per_t in part.send.items()}
        self.sendbuf = {peer: {t: torch.empty((len(idx), 4, d.ops[t].Np), dtype=dtype, device=dev)
                               for t, idx in per_t.items()}
                        for peer, per_t in part.send.items()}
        if isinstance(transport, LoopbackTransport):
            transport.steppers[part.rank] = self
        self._build_subsets()

    def halo_source(self):
        return self.eff

    def send_buffers(self):
        return [(peer, self.sendbuf[peer][t]) for peer in sorted(self.sendbuf)
                for t in self.disc.types if t in self.sendbuf[peer]]

    def recv_buffers(self, q):
        return [(peer, q[t][a:b]) for peer in sorted(self.part.recv)
                for t in self.disc.types if t in self.part.recv[peer]
                for a, b in [self.part.recv[peer][t]]]

    def receive_from(self, other, q):
        """Loopback: ghost rows copied from the owner's effective state."""
        src = other.halo_source()
        for t, (a, b) in self.part.recv[other.part.rank].items():
            q[t][a:b].copy_(src[t][other.send_idx[self.part.rank][t].long()])

    def _build_subsets(self):
        d, part, L = self.disc, self.part, self.L
        mesh = d.mesh
        dev = d.device
        names = ("hex", "wedge", "pyramid", "tet")
        owned = {t: np.arange(d.n_elems[t]) < part.n_owned[t] for t in d.types}
        sent = {t: np.zeros(d.n_elems[t], dtype=bool) for t in d.types}
        for per_t in part.send.values():
            for t, idx in per_t.items():
                sent[t][idx] = True
        # read set of level lev: its owned elements and their face neighbours
        need = {}
        for lev in range(1, L + 1):
            own = {t: owned[t] & (self.levels[t] == lev) for t in d.types}
            nd = {t: own[t].copy() for t in d.types}
            for t in d.types:
                nb = mesh.nbr[t][own[t]]
                for tid2, t2 in enumerate(names):
                    if t2 not in nd:
                        continue
                    sel = nb[:, :, 0] == tid2
                    nd[t2][nb[:, :, 1][sel]] = True
            need[lev] = nd
        empty = torch.zeros(0, dtype=torch.int32, device=dev)

        def sub(masks):
            lists = [empty] * 4
            for t in d.types:
                idx = np.flatnonzero(masks[t]).astype(np.int32)
                lists[TYPE_ID[t]] = torch.as_tensor(idx, device=dev) if len(idx) else empty
            self._keep.append(lists)
            self._ntypes[id(lists)] = sum(1 for x in lists if x.numel())
            return nat.subset(lists), sum(int(x.numel()) for x in lists)

        self._keep, self._ntypes, eff_types = [], {}, {}
        self.eff_sub, self.trace_sub, self.step_sub = {}, {}, {}
        for tick in range(2 ** (L - 1)):
            stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
            needed = {t: np.any([need[lev][t] for lev in stepping], axis=0) for t in d.types}
            self.trace_sub[tick] = sub(needed)[0]
            for lev in range(1, L + 1):
                m = {t: (owned[t] & (needed[t] | sent[t])) & (self.levels[t] == lev)
                     for t in d.types}
                st, n = sub(m)
                self.eff_sub[(tick, lev)] = st if n else None
                eff_types[(tick, lev)] = self._ntypes[id(self._keep[-1])]
        step_types = {}
        for lev in range(1, L + 1):
            st, n = sub({t: owned[t] & (self.levels[t] == lev) for t in d.types})
            self.step_sub[lev] = st if n else None
            step_types[lev] = self._ntypes[id(self._keep[-1])]
        # kernel launches per macro step (bench gpu_launches): dense output,
        # halo packs, traces (publishing types), stage kernels
        sem = d.formulation.kind == "SEM"
        pub = [t for t in d.types if t in (("wedge", "pyramid") if sem else ("hex", "wedge", "pyramid"))]
        npack = sum(len(per_t) for per_t in part.send.values())
        n = 0
        for tick in range(2 ** (L - 1)):
            stepping = [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]
            n += npack + len(pub) + sum(step_types[lev] for lev in stepping)
            # dense output: one multi-type launch per level with a subset
            n += sum(1 for lev in range(1, L + 1) if eff_types[(tick, lev)])
        self.launches_per_macro = n

    def _pack(self):
        L_, st, dm = nat.lib(), self.disc.stream_ptr(), self.disc.device_mesh
        for peer, per_t in self.send_idx.items():
            for t, idx in per_t.items():
                nat.check(L_.hw_halo_pack(dm.struct, TYPE_ID[t], self.eff[t].data_ptr(),
                                          idx.data_ptr(), idx.numel(),
                                          self.sendbuf[peer][t].data_ptr(), st))

    def _fields(self, s_):
        """HWFields of a persistent state dict (q, eff, ring slots), built
        once: the per-tick launches are bound by host overhead."""
        f = self._fcache.get(id(s_))
        if f is None:
            f = self._fcache[id(s_)] = (s_, nat.fields(self.disc.slots(s_)))
        return f[1]

    def tick_effective(self, tick, dt_min):
        """Dense output of this tick's owned read / sent elements, packed for
        the peers."""
        d, L = self.disc, self.L
        lib, dm, st = nat.lib(), d.device_mesh, d.stream_ptr()
        F = self._fields
        for lev in range(1, L + 1):
            sub = self.eff_sub[(tick, lev)]
            if sub is None:
                continue
            period = 2 ** (L - lev)
            frac = tick % period
            nh = self.n_hist[lev]
            if frac == 0 or nh == 0:
                nat.check(lib.hw_axpy3(dm.struct, F(self.q), F(self.eff), F(self.ring[0]), None,
                                       None, 1, 0.0, 0.0, 0.0, 0.0, sub, st))
                continue
            c = _dense_coeffs(nh, frac, period)
            s0 = self.steps[lev] % 3
            h = [self.ring[s0], self.ring[(s0 - 1) % 3], self.ring[(s0 - 2) % 3]]
            nat.check(lib.hw_axpy3(dm.struct, F(self.q), F(self.eff), F(h[0]), F(h[1]), F(h[2]),
                                   nh, c[0], c[1], c[2], dt_min * period, sub, st))
        self._pack()

    def tick_exchange(self):
        """Start the exchange of the packed boundary rows into the peers'
        ghost rows (returns the transport handle)."""
        return self.transport.start(self, self.eff)

    def tick_step(self, tick, dt_min, handle):
        """Wait for the ghosts' effective state, traces of the read set, and
        the fused RHS + AB3 update of the owned stepping elements."""
        d, L = self.disc, self.L
        lib, dm, st = nat.lib(), d.device_mesh, d.stream_ptr()
        F = self._fields
        self.transport.wait(handle)
        dm.compute_traces(F(self.eff), 0, st, subset=self.trace_sub[tick])
        dm.set_traces(0, None)
        if dm.corr:   # wedge face corrections from the effective state's traces (whole halo here)
            d.apply_corrections()
        for lev in [lev for lev in range(1, L + 1) if tick % (2 ** (L - lev)) == 0]:
            self.n_hist[lev] = min(self.n_hist[lev] + 1, 3)
            self.steps[lev] += 1
            sub = self.step_sub[lev]
            if sub is None:
                continue
            s0 = self.steps[lev] % 3
            h0, h1, h2 = self.ring[s0], self.ring[(s0 - 1) % 3], self.ring[(s0 - 2) % 3]
            nh = self.n_hist[lev]
            c = _ab_coeffs(nh)
            nat.check(lib.hw_ab_step(dm.struct, F(self.eff), F(self.q), F(h0), F(h1), F(h2), nh,
                                     c[0], c[1], c[2], dt_min * 2 ** (L - lev), sub, st))

    def macro_step(self, dt_min):
        for tick in range(2 ** (self.L - 1)):
            self.tick_effective(tick, dt_min)
            self.tick_step(tick, dt_min, self.tick_exchange())

    def owned_state(self):
        return {t: self.q[t][:self.part.n_owned[t]] for t in self.disc.types}
